#!/bin/bash
# Launch list (ncu gpu__time_duration per launch) + optional full captures of
# the kernels named in $NCU_KERNELS, for the default bench workload.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/build.log; exit 1; }
Q="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-secondary --no-explorer ${BENCH_ARGS}"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches.csv python bench.py $Q > gpurun_out/ncu_launch_run.log 2>&1; echo "ncu_launches=$?"
python -c "import sys; sys.path.insert(0, \"tools\"); import ncu_summary as n; print(n.launches(\"gpurun_out/launches.csv\"))"
for k in ${NCU_KERNELS}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${k}_kernel -s 7 -c 1 -o gpurun_out/prof_${k} -f python bench.py $Q > gpurun_out/ncu_${k}.log 2>&1; echo "ncu_${k}=$?"
done
