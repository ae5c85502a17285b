#!/bin/bash
# A/B of the C5 NTT sweep for experimental library builds (exp/libsecn_*.so) against the in-tree one.
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
cp paper_2506_11586_b200/libsecn.so /tmp/libsecn_base.so
run() {
  timeout 300 python bench.py --net ntt_sweep --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
rows=d.get('ntt_sweep') or d.get('sweep') or []
for r in rows:
    if r['L']==4 and r['word_bits']==32: print('  N=%d fwd %.1fM/s (%.2f) inv %.1fM/s (%.2f)'%(r['N'],r['fwd_ntt_per_s']/1e6,r['fwd_hbm_frac'],r['inv_ntt_per_s']/1e6,r['inv_hbm_frac']))
"
}
echo "== base"; run
for v in "$@"; do
  cp exp/libsecn_$v.so paper_2506_11586_b200/libsecn.so; touch paper_2506_11586_b200/libsecn.so
  echo "== $v"; run
done
cp /tmp/libsecn_base.so paper_2506_11586_b200/libsecn.so
