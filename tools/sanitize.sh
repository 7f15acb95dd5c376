#!/bin/bash
# compute-sanitizer pass on the GPU box (dev tool): memcheck, racecheck and
# synccheck over smoke() and a larger stencil + classified tree-reduction run.
python -c "import __graft_entry__ as g; g.build()" || exit 1
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 6 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | grep -v "Host Frame" | tail -4
  timeout 1500 compute-sanitizer --tool $tool --print-limit 6 python tools/sanitize_workload.py 2>&1 | grep -v "Host Frame" | tail -4
done
