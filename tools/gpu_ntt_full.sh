#!/bin/bash
# ncu --set full (with source) of the batched forward and inverse NTT of the C5 sweep at one ring
# degree (32-bit limbs, 256 MiB per call), plus the shared-memory bank-conflict counters; per
# kernel summary (tools/ncu_summary.py) and per-SASS-op stall breakdown (tools/ncu_stalls.py).
# Usage: tools/gpu_ntt_full.sh TAG [log_n]   (outputs in gpurun_out/)
set -u
O=gpurun_out; mkdir -p $O
TAG=${1:-cur}; LOGN=${2:-12}
python -c "import __graft_entry__ as g; g.build()" > $O/build_nttfull.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python tools/sweep_profile.py 32 256 $LOGN > $O/ntt_full_$TAG.log 2>&1 || { echo sweep_profile failed; tail $O/ntt_full_$TAG.log; exit 1; }
SM="l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum"
for d in fwd inv; do
  SKIP=0; [ $d = inv ] && SKIP=1
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none --metrics $SM \
    --launch-skip $SKIP --launch-count 1 -f -o $O/ntt_full_${TAG}_$d python tools/sweep_profile.py 32 256 $LOGN >> $O/ntt_full_$TAG.log 2>&1
  echo "ncu $d rc=$?"
  { python tools/ncu_summary.py $O/ntt_full_${TAG}_$d.ncu-rep; python tools/ncu_stalls.py $O/ntt_full_${TAG}_$d.ncu-rep k_ntt;
    ncu -i $O/ntt_full_${TAG}_$d.ncu-rep --page raw --csv --metrics $SM,launch__registers_per_thread,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers; } >> $O/ntt_full_${TAG}_summary.txt 2>&1
done
cat $O/ntt_full_${TAG}_summary.txt
