mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
for rep in 1 2; do
for v in 1776 445 600 800 1000; do
  SECN_NTT_NP2_MIN=$v timeout 300 python bench.py --steps 200 --warmup 5 --no-e2e --no-online --no-companion --no-sweep --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('NP2_MIN=$v', d['ms_per_step'], d['roofline']['stage_ms'])"
done; done
SWEEP=1 timeout 300 python tools/variant_sweep.py squeezenet1_1 'SECN_NTT_NP2_MIN=1776' 'SECN_NTT_NP2_MIN=445' 'SECN_NTT_NP2_MIN=2' 2>&1 | tail -30
