#!/bin/bash
# A/B the librc build flags on the GPU box: tools/ab.sh "<flagsA>" "<flagsB>" ... (dev tool)
for f in "$@"; do
  RC_EXTRA_NVCC_FLAGS="$f" python -c "from paper_1308_3203_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  echo "== flags [$f]"
  python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],3), 'Gaccess/s', round(d['ms_per_step'],1), 'ms')
k=d.get('kernels') or {}
print('  ', {a:round(v['ms_per_step'],1) for a,v in k.items() if isinstance(v,dict) and v['ms_per_step']>1})"
done
