#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build_fin.log 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_fin.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_fin.log
for o in free staged none; do OVERLAP=$o REPS=50 timeout 400 python tools/staged_stress.py > $O/stress_$o.txt 2>&1; echo "stress: $(tail -1 $O/stress_$o.txt)"; done
for i in 1 2 3; do echo "online_check free: $(timeout 200 python tools/online_check.py 2>&1 | grep mismatches | tr '\n' ' ')"; done
timeout 300 python bench.py --net resnet50 --steps 10 --warmup 3 --no-companion --no-cpu-baseline --no-e2e --no-online --no-sweep > $O/bench_r50.json 2>/dev/null; python -c "import json;d=json.loads(open('$O/bench_r50.json').read().strip().splitlines()[-1]);print('R50',d['ms_per_step'])"
