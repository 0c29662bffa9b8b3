#!/bin/bash
# A/B sweep timings of library variants on the GPU box:
#   tools/ab.sh "2d5:2048,2d5:4096" libsrj.so libsrj_x.so ...   (env SKEW=0|1, LEVEL, SPP)
cases=$1; shift
for lib in "$@"; do
  echo "== $lib"
  SRJ_LIBRARY=$PWD/paper_2011_06636_b200/$lib SRJ_TB_SKEW=${SKEW:-1} python tools/sweep_bench.py "$cases" --level ${LEVEL:-14} --spp ${SPP:-6} 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print('  %-10s %8.3f us/sweep %7.1f GLUP/s'%(d['case'],d['us_per_sweep'],d['GLUPs']))
    except Exception: print(l.rstrip()[:200])
"
done
