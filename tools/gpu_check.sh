#!/bin/bash
# GPU-box check after a change (dev tool): build + smoke, GPU tests, A/B bench
# of the given build flags (default: the plain build).
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
if [ $# -eq 0 ]; then bash tools/ab.sh ""; else bash tools/ab.sh "$@"; fi
