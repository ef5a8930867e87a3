# 16-bit storage on the staged row kernel (f32 fold) vs the per-thread loop nest
P="python scripts/r02/generic_probe.py"
for env in "BGX_NO_ROWREDUCE=1" "BGX_X=1"; do
  echo "== $env"
  env $env $P "(c,a,b)->(a,c)" a=256,c=4096,b=64 auto bfloat16
  env $env $P "(i,k)->(i)" i=65536,k=512 auto bfloat16
  env $env $P "(i,k),(k)->(i)" i=65536,k=512 auto bfloat16
  env $env $P "(i,k),(i,k)->(i)" i=32768,k=768 auto float16
  env $env $P "(a,d,c),(a),(a)->(a,d)" a=4096,d=64,c=64 auto bfloat16
done
