for env in "" "BGX_RR_WIDE=1"; do
  echo "== ${env:-4-warp 32-column tiles}"
  for s in "(i,k)->(i) i=65536,k=1024" "(i,k)->(i) i=32768,k=4096" "(i,k)->(i) i=262144,k=256" "(i,k)->(i) i=20000,k=96" "(i,j,k)->(i,j) i=256,j=256,k=512"; do
    set -- $s; env $env python scripts/r02/generic_probe.py "$1" "$2"
  done
done
