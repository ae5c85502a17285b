python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py --no-sweep --no-online --batched-leg 0 --no-e2e --no-cpu-baseline --steps 50 > gpurun_out/bench_r02w_alu.json 2> gpurun_out/bench_r02w_alu.err; echo "alu rc=$?"
timeout 900 python bench.py --net squeezenet1_0 --steps 50 --no-sweep --batched-leg 0 --no-companion > gpurun_out/bench_r02w_sq10.json 2> gpurun_out/bench_r02w_sq10.err; echo "sq10 rc=$?"
timeout 1200 python bench.py --net resnet50 --steps 20 --no-sweep --batched-leg 0 --no-companion > gpurun_out/bench_r02w_r50.json 2> gpurun_out/bench_r02w_r50.err; echo "r50 rc=$?"
bash tools/gpu_step_ncu.sh r02w > /dev/null 2>&1; echo "stepncu rc=$?"
bash tools/gpu_step_ncu_w64.sh r02w64 > /dev/null 2>&1; echo "stepncu64 rc=$?"
rm -f gpurun_out/*.ncu-rep
