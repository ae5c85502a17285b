#!/bin/bash
# A/B timing of an experimental library build (exp/libsecn_*.so) against the in-tree one.
set -u
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
cp paper_2506_11586_b200/libsecn.so /tmp/libsecn_base.so
run() {
  timeout 200 python tools/ntt_time.py 8192 2>&1 | tail -2
  timeout 300 python bench.py --steps 30 --warmup 5 --no-companion --no-cpu-baseline --no-e2e --no-online --no-sweep > $O/bench_exp.json 2>/dev/null
  python -c "import json;d=json.loads(open('$O/bench_exp.json').read().strip().splitlines()[-1]);print('STEP_MS',d['ms_per_step'],d['roofline']['stage_ms'])"
}
echo "== base"; run
for v in "$@"; do
  cp exp/libsecn_$v.so paper_2506_11586_b200/libsecn.so; touch paper_2506_11586_b200/libsecn.so
  echo "== $v"; run
done
cp /tmp/libsecn_base.so paper_2506_11586_b200/libsecn.so
