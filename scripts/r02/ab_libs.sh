# same probe against several builds, interleaved twice: bash ab_libs.sh VARS shapes... -- libs...
V=$1; shift
SH=""; while [ "$1" != "--" ]; do SH="$SH $1"; shift; done; shift
for rep in 1 2; do
for L in "$@"; do
  echo "== $L rep $rep"
  if [ "$L" = base ]; then VARS=$V python scripts/r02/probe_drain.py $SH
  else BGX_LIB=$PWD/paper_2503_04771_b200/libbgx_$L.so VARS=$V python scripts/r02/probe_drain.py $SH; fi
done; done
