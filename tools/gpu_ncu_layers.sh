#!/bin/bash
# ncu --set full (with source) of every kernel of single layers on the bench step's path (device
# mask encoded ahead, secn32_he_conv2d_em): k_mask_encode, forward NTT, MAC, INTT tail.
# Usage: tools/gpu_ncu_layers.sh TAG layer...   (outputs in gpurun_out/ncu_TAG_<layer>.ncu-rep)
set -u
O=gpurun_out; mkdir -p $O
TAG=$1; shift
python -c "import __graft_entry__ as g; g.build()" > $O/build_ncu.log 2>&1 || { echo build failed; exit 1; }
for L in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on --launch-skip 8 --launch-count 4 \
    -f -o $O/ncu_${TAG}_$L python tools/prof_layer.py $L squeezenet1_1 3 32 em > $O/ncu_${TAG}_$L.log 2>&1
  echo "ncu $L rc=$?"
done
