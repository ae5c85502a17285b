#!/bin/bash
# Quick GPU check: build, GPU tests (optionally filtered), per-layer times, bench without the CPU legs.
set -u
O=gpurun_out; mkdir -p $O
TAG=${1:-q}; K=${2:-}
python -c "import __graft_entry__ as g; g.build()" > $O/build_$TAG.log 2>&1 || { echo build failed; tail -20 $O/build_$TAG.log; exit 1; }
if [ -n "$K" ]; then timeout 600 python -m pytest tests -m gpu -x -q -k "$K" > $O/pytest_$TAG.log 2>&1; else timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_$TAG.log 2>&1; fi
echo "pytest rc=$?"; tail -5 $O/pytest_$TAG.log
timeout 300 python tools/layer_times.py 32 > $O/layer_times_$TAG.txt 2>&1; echo "layer_times rc=$?"; tail -30 $O/layer_times_$TAG.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-companion --no-cpu-baseline --no-e2e --no-online --no-sweep > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$O/bench_$TAG.json').read().strip().splitlines()[-1]);print('STEP_MS',d['ms_per_step'],d['roofline'])"
