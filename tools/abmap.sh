#!/bin/bash
# A/B helper: variant libraries live in tools/scratch/<name>/ (git-ignored, built by tools/mkvar.sh)
# mapping numbers (sliding_ba it/s, map_step it/s) of bench.py against each variant library
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
for v in "$@"; do
  GSF_LIB=$PWD/tools/scratch/$v/libgsf_cuda.so timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/abm_$v.json 2> gpurun_out/abm_$v.err
  python - "$v" <<'PY'
import json,sys
v=sys.argv[1]
try:
  d=json.loads(open(f"gpurun_out/abm_{v}.json").read().strip().splitlines()[-1]); m=d['mapping']
  k=m.get('kernels',{})
  print(v, 'track', round(d['value'],3), 'sliding_ba', round(m['value'],2), 'it/s', round(m['ms_per_iter'],3), 'ms  map_step', round(m['map_step_it_per_s'],1),
        ' '.join(f"{n}={k[n]['avg_ms']*1e3:.1f}" for n in k if isinstance(k[n], dict)))
except Exception as e: print(v,'FAILED',e)
PY
done
