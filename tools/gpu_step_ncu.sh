#!/bin/bash
# ncu of every kernel of one bench step (tools/step_profile.py), with DRAM bytes, instructions,
# pipe utilisation and stall reasons; summarised by tools/ncu_step_summary.py. Outputs in gpurun_out/.
set -u
O=gpurun_out; mkdir -p $O
TAG=${1:-cur}
python -c "import __graft_entry__ as g; g.build()" > $O/build_stepncu.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python tools/step_profile.py > $O/step_profile_$TAG.log 2>&1 || { echo step_profile failed; tail $O/step_profile_$TAG.log; exit 1; }
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum"
M="$M,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"
M="$M,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active"
M="$M,dram__throughput.avg.pct_of_peak_sustained_elapsed"
M="$M,smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct,smsp__sass_average_data_bytes_per_sector_mem_global_op_st.pct"
M="$M,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"
for s in wait long_scoreboard short_scoreboard math_pipe_throttle barrier membar not_selected selected dispatch_stall no_instruction mio_throttle lg_throttle sleeping branch_resolving drain tex_throttle imc_miss misc; do
  M="$M,smsp__average_warps_issue_stalled_${s}_per_issue_active.ratio"
done
timeout 1200 ncu --profile-from-start off --clock-control none --metrics $M -f -o $O/step_$TAG python tools/step_profile.py > $O/step_ncu_$TAG.log 2>&1
echo "ncu rc=$?"
python tools/ncu_step_summary.py $O/step_$TAG.ncu-rep $O/${TAG}_step_ncu.json > $O/step_summary_$TAG.txt 2>&1; cat $O/step_summary_$TAG.txt
