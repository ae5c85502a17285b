#!/bin/bash
# ncu --set full of the three kernels of two small SqueezeNet layers (fire2.e1, fire9.e3)
set -u
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build_ncu.log 2>&1 || { echo build failed; exit 1; }
for L in fire2.e1 fire9.e3; do
  timeout 300 python tools/prof_layer.py $L squeezenet1_1 2 32 || exit 1
  timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_mac|k_ntt_inv_tail2|k_ntt_fwd' \
    --launch-skip 3 --launch-count 3 -f -o $O/ncu_$L python tools/prof_layer.py $L squeezenet1_1 2 32 > $O/ncu_$L.log 2>&1
  echo "ncu $L rc=$?"
done
