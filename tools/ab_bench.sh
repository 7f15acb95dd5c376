#!/bin/bash
# dev tool: A/B the bench over librc variants built with extra nvcc flags.
#   tools/ab_bench.sh out_prefix "" "-DLS_NB=3" ...   (variant 0 = default flags)
# Each variant: rebuild in-tree, short bench (main line only), JSON to
# gpurun_out/<prefix>_<i>.json; the default build is restored at the end.
prefix=$1; shift
i=0
for flags in "$@"; do
  RC_EXTRA_NVCC_FLAGS="$flags" python -c "from paper_1308_3203_b200 import _build; _build.build()" || exit 1
  python bench.py --steps ${AB_STEPS:-5} --warmup 3 --no-secondary --no-explorer --no-cpu-baseline --no-e2e \
    > gpurun_out/${prefix}_$i.json 2> gpurun_out/${prefix}_$i.err
  echo "variant $i [$flags]: $(python -c "import json; d=json.load(open('gpurun_out/${prefix}_$i.json')); k=d['kernels']; print(round(d['value'],2), {c: round(k[c]['ms_per_step'],1) for c in ('interp','filter','sort','detect')})")"
  i=$((i+1))
done
python -c "from paper_1308_3203_b200 import _build; _build.build()"
