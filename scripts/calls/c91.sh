#!/bin/bash
for v in on off on off; do
  if [ $v = off ]; then export BGX_SIMT_KT256_OFF=1; else unset BGX_SIMT_KT256_OFF; fi
  echo "== KT256 $v"; python scripts/overhead.py 2>&1 | grep "256, 256"
done
python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_golden.py -x -q 2>&1 | tail -1
