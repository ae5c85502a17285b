#!/bin/bash
# One gpurun call: GPU tests, the default bench line, per-layer times, the ncu launch list of the
# bench step and one ncu --set full capture of conv10 (the dominant layer). Outputs in gpurun_out/.
set -u
O=gpurun_out; mkdir -p $O
TAG=${1:-cur}
python -c "import __graft_entry__ as g; g.build()" > $O/build_$TAG.log 2>&1 || { echo build failed; exit 1; }
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" | tee -a $O/pytest_gpu_$TAG.log
fi
timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?"
tail -c 3000 $O/bench_$TAG.json
timeout 600 python tools/layer_times.py 32 > $O/layer_times_$TAG.txt 2>&1; echo "layer_times rc=$?"
if [ "${SKIP_NCU:-0}" != 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-companion --no-cpu-baseline --no-e2e --no-online --no-sweep --batched-leg 0 > $O/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mac -c 1 -f -o $O/conv10_$TAG \
    python tools/prof_layer.py conv10 squeezenet1_1 2 32 > $O/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
fi
timeout 300 python tools/trace_step.py squeezenet1_1 32 > $O/trace_step_$TAG.txt 2>&1; echo "trace rc=$?"; tail -3 $O/trace_step_$TAG.txt
python tools/ncu_summary.py $O/conv10_$TAG.ncu-rep > $O/conv10_summary_$TAG.txt 2>&1; python tools/kmac_traffic.py $O/conv10_$TAG.ncu-rep "profiles/${TAG}_ncu_conv10_kmac_summary.txt (ncu --set full --clock-control none, tools/prof_layer.py conv10 squeezenet1_1 2 32)" > $O/kmac_traffic_$TAG.log 2>&1; cp profiles/kmac_traffic.json $O/kmac_traffic_$TAG.json
