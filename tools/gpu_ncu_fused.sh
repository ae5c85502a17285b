set -u
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build_ncu.log 2>&1 || { echo build failed; exit 1; }
L=fire9.e3
SECN_FUSED=0 timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_mac|k_ntt_inv_tail2' \
    --launch-skip 4 --launch-count 2 -f -o $O/ncu_f0_$L python tools/prof_layer.py $L squeezenet1_1 2 32 > $O/ncu_f0_$L.log 2>&1
echo "f0 rc=$?"
SECN_FUSED=2 SECN_FUSED_SG=1 SECN_FUSED_MT=1 timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_layer_fused' \
    --launch-skip 2 --launch-count 1 -f -o $O/ncu_f11_$L python tools/prof_layer.py $L squeezenet1_1 2 32 > $O/ncu_f11_$L.log 2>&1
echo "f11 rc=$?"
SECN_FUSED=2 SECN_FUSED_SG=1 SECN_FUSED_MT=2 timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_layer_fused' \
    --launch-skip 2 --launch-count 1 -f -o $O/ncu_f12_$L python tools/prof_layer.py $L squeezenet1_1 2 32 > $O/ncu_f12_$L.log 2>&1
echo "f12 rc=$?"
