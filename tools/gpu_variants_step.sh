#!/bin/bash
# The bench step (with the 64-bit companion), the C5 sweep and a parity subset under alternative
# builds of libsecn.so (variants/*.so, built here with extra -D flags; git-ignored, shipped by
# gpurun) -> gpurun_out/{step,sweep,pt}_<variant>.*; the default build is restored at the end.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2506_11586_b200/libsecn.so /tmp/libsecn_default.so
for v in variants/*.so; do
  n=$(basename $v .so)
  cp $v paper_2506_11586_b200/libsecn.so; touch paper_2506_11586_b200/libsecn.so
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mask.py -q -x -k "ntt or tiny or shapes or mask or gen" > gpurun_out/pt_$n.log 2>&1
  for i in 1 2; do
    timeout 600 python bench.py --no-sweep --no-cpu-baseline --no-online --no-e2e --batched-leg 0 > gpurun_out/step_${n}_$i.json 2> /dev/null
  done
  timeout 600 python bench.py --net ntt_sweep --steps 10 > gpurun_out/sweep_$n.json 2> /dev/null
done
cp /tmp/libsecn_default.so paper_2506_11586_b200/libsecn.so
