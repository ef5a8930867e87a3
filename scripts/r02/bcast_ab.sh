# broadcast elementwise: row-per-warp decode vs per-vector decode
P="python scripts/r02/generic_probe.py"
for env in "BGX_BCAST_NO_ROWS=1" "BGX_X=1"; do
  echo "== $env"
  env $env $P "(c,b,a),(b)->(c,b,a)" c=64,b=1024,a=1024
  env $env $P "(c),(a,c),(b)->(c,a,b)" c=8,a=1024,b=4096
  env $env $P "(c),(a,c),(b)->(c,a,b)" c=8,a=1024,b=4096 auto bfloat16
  env $env $P "(a,b),(b)->(a,b)" a=4096,b=8192
  env $env $P "(a),(b)->(a,b)" a=4096,b=8192
  env $env $P "(d,c,a),(c)->(d,c,a)" d=4096,c=8,a=256
done
