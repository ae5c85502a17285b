#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_ntt_fwd|k_ntt_inv' \
  --launch-skip 0 --launch-count 2 -f -o $O/ncu_ntt python tools/prof_ntt.py 32 4096 > $O/ncu_ntt.log 2>&1
echo "ncu rc=$?"
