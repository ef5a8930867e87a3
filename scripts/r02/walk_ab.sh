for env in "" "BGX_NO_WALK_ORDER=1"; do
  echo "== ${env:-walk order}"
  env $env python scripts/r02/generic_probe.py "(d,a,c),(c,d,b)->(b,c,d)" b=1024,c=64,d=1024,a=256
  env $env python scripts/r02/generic_probe.py "(d,b,a),(c,d,b)->(a,b,d)" a=1024,b=8,d=4096,c=64
  env $env python scripts/r02/generic_probe.py "(c),(d,c,b),(d,b,a)->(a,d)" a=64,d=1024,c=8,b=256
  env $env python scripts/r02/generic_probe.py "(a,b,c),(b)->(c,b,a)" c=64,b=1024,a=1024
done
