#!/bin/bash
for lib in paper_2503_04771_b200/libbgx.so oldlib/libbgx.so paper_2503_04771_b200/libbgx.so oldlib/libbgx.so; do
  echo "== $lib"; BGX_PROBE_LIB=$lib python scripts/rs_probe.py 2>&1 | tail -3 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print({k:(round(v,4) if isinstance(v,float) else v) for k,v in d.items() if k.startswith('ms')})"
done
