for env in "" "BGX_NO_ROWREDUCE=1"; do
  echo "== ${env:-rowreduce}"
  env $env python scripts/r02/generic_probe.py "(a,d,c),(b)->(d,a,c)" a=1024,d=1024,c=64,b=64
  env $env python scripts/r02/generic_probe.py "(b,c)->(c)" b=4096,c=4096
  env $env python scripts/r02/generic_probe.py "(b,c)->(c)" b=65536,c=256
  env $env python scripts/r02/generic_probe.py "(b,c)->(c)" b=256,c=65536
  env $env python scripts/r02/generic_probe.py "(b,c)->(c)" b=64,c=1048576
  env $env python scripts/r02/generic_probe.py "(b,c),(b)->(c)" b=4096,c=4096
  env $env python scripts/r02/generic_probe.py "(b,c),(b)->(c)" b=128,c=262144
  env $env python scripts/r02/generic_probe.py "(d,a,b),(b)->(b,d)" d=256,a=1024,b=256
  env $env python scripts/r02/generic_probe.py "(c,a,b)->(a,c)" a=256,c=4096,b=64
done
