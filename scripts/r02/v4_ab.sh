for env in "" "BGX_NO_GENERIC_V4=1"; do
  echo "== ${env:-four outputs per thread}"
  for s in "(i,k),(k,j),(j,l)->(i,l) i=256,k=256,j=256,l=256" "(i,k),(k,j),(j,l)->(i,l) i=512,k=128,j=128,l=512" "(d,a,c),(c,d,b)->(b,c,d) b=1024,c=64,d=1024,a=256" "(d,b,a),(c,d,b)->(a,b,d) a=1024,b=8,d=4096,c=64" "(a,d,c),(b)->(d,a,c) a=1024,d=1024,c=64,b=64" "(b,i,k),(b,k,j)->(b,i,j) b=64,i=64,k=64,j=256"; do
    set -- $s; env $env python scripts/r02/generic_probe.py "$1" "$2" exact
  done
done
