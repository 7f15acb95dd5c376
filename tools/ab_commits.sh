#!/bin/bash
# Same-box A/B of the working tree against older commits checked out (and
# built) under _ab/<name> (git worktrees, not committed): short bench lines.
Q="--steps ${STEPS:-5} --warmup 3 --no-secondary --no-explorer --no-cpu-baseline --no-e2e"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
  for d in . $(ls _ab 2>/dev/null | sed 's#^#_ab/#') ${VARIANTS}; do
    v=""; case "$d" in *=*) v="$d"; d=.;; esac
    (cd $d && env $v timeout 600 python bench.py $Q > /tmp/abq.json 2> /tmp/abq.err; echo "$d $v rep$rep: $(python -c "
import json; d=json.load(open('/tmp/abq.json')); k=d['kernels']
print(round(d['value'],2), round(d['ms_per_step'],1), {c: round(k[c]['ms_per_step'],1) for c in ('interp','sort','detect')})" 2>&1 | tail -1)")
  done
done
