# block-per-output chains for reductions the loop nest cannot coalesce
P="python scripts/r02/generic_probe.py"
for env in "BGX_NO_CG_WIDE=1" "BGX_X=1"; do
  echo "== $env"
  env $env $P "(d,a,c),(c,a),(c)->(d)" d=4096,a=8,c=256
  env $env $P "(a,b,c),(c,b)->(a)" a=8192,b=32,c=64
  env $env $P "(a,b,c),(c,b)->(a)" a=32768,b=8,c=32
  env $env $P "(a,b,c),(c,b)->(a)" a=16384,b=16,c=64 auto float64
  env $env $P "(c),(c,a,d)->(c,a)" c=256,a=256,d=256
  env $env $P "(b,a,c),(c,a)->(b)" b=2048,a=64,c=64
  env $env $P "(x,a,c),(c,a)->(x)" x=30000,a=16,c=16
done
