#!/bin/bash
# bench step time (graph) under several settings of the libsecn tuning knobs; two passes.
# Usage: bash tools/gpu_knob_sweep.sh 'A=1 B=2' 'A=3' ...
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
for rep in 1 2; do
for v in "$@"; do
  env $v timeout 300 python bench.py --steps 200 --warmup 5 --no-e2e --no-online --no-companion --no-sweep --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v'.ljust(28), d['ms_per_step'], d['roofline']['frac'])"
done; done
