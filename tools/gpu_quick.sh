#!/bin/bash
# Quick GPU-box pass: smoke, the fast gpu tests, and short bench A/B lines
# (default path vs the env variants given as arguments, e.g. RC_SORT_LSD=1).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"; tail -3 gpurun_out/smoke.log
if [ "${TESTS:-1}" != "0" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "not slow" ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1; echo "tests=$?"; tail -15 gpurun_out/gpu_tests.log
fi
Q="--steps ${STEPS:-5} --warmup 3 --no-secondary --no-explorer --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
i=0
for v in "" "$@"; do
  env $v timeout 600 python bench.py $Q > gpurun_out/quick_$i.json 2> gpurun_out/quick_$i.err
  echo "variant $i [$v] rc=$?: $(python -c "
import json; d=json.load(open('gpurun_out/quick_$i.json')); k=d['kernels']
print(round(d['value'],2), round(d['ms_per_step'],1), {c: round(k[c]['ms_per_step'],1) for c in ('interp','filter','sort','detect')})" 2>&1 | tail -1)"
  i=$((i+1))
done
