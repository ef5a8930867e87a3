for tj in 32 64 128; do
  echo "== thin tile columns $tj"
  for s in "(i,k),(k)->(i) i=8192,k=8192" "(i,k)->(i) i=8192,k=8192" "(i,k),(k)->(i) i=2048,k=65536" "(i,k),(i,k)->(i) i=4096,k=16384" "(i,k)->(i) i=700,k=4096" "(i,k),(k)->(i) i=4096,k=1000"; do
    set -- $s; BGX_RR_THIN_TJ=$tj python scripts/r02/generic_probe.py "$1" "$2"
  done
done
