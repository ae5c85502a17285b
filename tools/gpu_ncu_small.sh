#!/bin/bash
# ncu --set full (with source counters) of the MAC and tail kernels of small SqueezeNet layers
# (fire4.e1: k_mac_ws; fire9.e3: k_mac), one launch each. Outputs in gpurun_out/.
set -u
O=gpurun_out; mkdir -p $O
TAG=${1:-cur}
python -c "import __graft_entry__ as g; g.build()" > $O/build_ncu.log 2>&1 || { echo build failed; exit 1; }
for L in fire4.e1 fire9.e3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_mac|k_ntt_inv_tail2' \
    --launch-skip 2 --launch-count 2 -f -o $O/ncu_${TAG}_$L python tools/prof_layer.py $L squeezenet1_1 2 32 > $O/ncu_${TAG}_$L.log 2>&1
  echo "ncu $L rc=$?"
done
