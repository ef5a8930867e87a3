# tolerance-mode (tree) reductions with and without axis coalescing
P="python scripts/r02/generic_probe.py"
for env in "BGX_NO_COALESCE=1" "BGX_X=1"; do
  echo "== $env"
  env $env $P "(d,b,a)->(a)" a=1024,d=1024,b=8 auto bfloat16
  env $env $P "(d,b,a)->(d)" d=256,b=256,a=64 auto bfloat16
  env $env $P "(d,b,a)->(a)" a=1024,d=1024,b=8 ffma
  env $env $P "(a,b,c,d)->(a)" a=64,b=64,c=64,d=64 ffma
  env $env $P "(a,b,c,d)->(d)" a=64,b=64,c=64,d=64 ffma
  env $env $P "(c,a,b),(b,c)->()" c=8,a=256,b=4096 auto bfloat16
  env $env $P "(a,c)->()" a=4096,c=1024 auto bfloat16
done
