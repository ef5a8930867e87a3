# exact column chains after the issue-in-the-add-shadow reorder: CPW 8 vs 32
P="python scripts/r02/generic_probe.py"
for env in "BGX_X=1" "BGX_CC_CPW=32" "BGX_CC_CPW=8"; do
  echo "== $env"
  env $env $P "(k,i),(k)->(i)" k=8192,i=8192
  env $env $P "(k,i),(k)->(i)" k=8192,i=8192 auto float64
  env $env $P "(b,k,i),(b,k)->(b,i)" b=64,k=1024,i=1024
  env $env $P "(i,k)->(k)" i=8192,k=8192
  env $env $P "(b,c),(b)->(c)" b=128,c=262144
  env $env $P "(b,c)->(c)" b=4096,c=4096
  env $env $P "(b,c)->(c)" b=16384,c=1024
  env $env $P "(b,c),(b)->(c)" b=16384,c=1024
  env $env $P "(b,c)->(c)" b=32768,c=512
  env $env $P "(b,c)->(c)" b=32768,c=512 auto float64
  env $env $P "(k,i),(k,i)->(i)" k=4096,i=8192
done
