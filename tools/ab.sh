#!/bin/bash
# A/B helper: variant libraries live in tools/scratch/<name>/ (git-ignored, built by tools/mkvar.sh)
# run the bench (tracking only) against each variant library; one summary line per variant
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
for v in "$@"; do
  GSF_LIB=$PWD/tools/scratch/$v/libgsf_cuda.so timeout 300 python bench.py --no-mapping --no-cpu-baseline > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python - "$v" <<'PY'
import json,sys
v=sys.argv[1]
try:
  d=json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
  k=d['kernels']; print(v, round(d['value'],3), 'it_ms', round(d['ms_per_iter']*1e3,1), ' '.join(f"{n}={k[n]['avg_ms']*1e3:.1f}" for n in k if isinstance(k[n], dict)))
except Exception as e: print(v,'FAILED',e)
PY
done
