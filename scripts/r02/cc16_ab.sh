# 16-bit storage on the column-chain kernel vs the loop nest; f32 regression check
P="python scripts/r02/generic_probe.py"
for env in "BGX_NO_COLCHAIN=1" "BGX_X=1"; do
  echo "== $env"
  env $env $P "(k,i)->(i)" k=512,i=65536 auto bfloat16
  env $env $P "(k,i),(k,i)->(i)" k=768,i=32768 auto float16
  env $env $P "(a,b,d)->(b,d)" a=64,b=1024,d=64 auto bfloat16
  env $env $P "(k,i),(k)->(i)" k=8192,i=8192
  env $env $P "(i,k)->(k)" i=8192,k=8192
done
for env in "BGX_NO_COLCHAIN=1" "BGX_X=1"; do
  echo "== shared vector, $env"
  env $env $P "(k,i),(k)->(i)" k=768,i=32768 auto bfloat16
  env $env $P "(b,k,i),(b,k)->(b,i)" b=64,k=512,i=1024 auto bfloat16
done
