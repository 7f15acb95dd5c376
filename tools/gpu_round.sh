#!/bin/bash
# One GPU-box pass: build + smoke, GPU tests, ncu launch list and full
# captures of the top kernels (summarised on the box so bench.py's roofline
# `traffic` comes from this code's capture), then the bench line.  Env
# switches: TESTS=0/1/fast BENCH=0/1 NCU=0/1 BENCH_ARGS="..." (extra bench.py
# args).  Everything lands in gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"; tail -2 gpurun_out/smoke.log
if [ "${TESTS:-1}" != "0" ]; then
  K=""; [ "${TESTS}" == "fast" ] && K='-k "not slow"'
  eval timeout 2000 python -m pytest tests -m gpu -x -q $K > gpurun_out/gpu_tests.log 2>&1; echo "tests=$?"; tail -4 gpurun_out/gpu_tests.log
fi
if [ "${NCU:-1}" != "0" ]; then
  Q="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline ${BENCH_ARGS}"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches.csv python bench.py $Q > gpurun_out/ncu_launch_run.log 2>&1; echo "ncu_launches=$?"
  for k in ${NCU_KERNELS:-k1c bucket_detect}; do
    re="${k}_kernel"; [ "$k" == "k1c" ] && re="rc_k1c"
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:${re} -s 7 -c 1 -o gpurun_out/prof_${k} -f python bench.py $Q > gpurun_out/ncu_${k}.log 2>&1; echo "ncu_${k}=$?"
  done
  python tools/ncu_summary.py --round box --tag tmp > /dev/null 2>&1  # profiles/ncu_traffic.json for the bench below
fi
if [ "${BENCH:-1}" != "0" ]; then
  timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
fi
