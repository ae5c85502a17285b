#!/bin/bash
# ResNet-50 and SqueezeNet-1.0 bench lines under every variants/*.so build (see gpu_variants.sh)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2506_11586_b200/libsecn.so /tmp/libsecn_default.so
for v in variants/*.so; do
  n=$(basename $v .so)
  cp $v paper_2506_11586_b200/libsecn.so; touch paper_2506_11586_b200/libsecn.so
  timeout 900 python bench.py --net resnet50 --steps 10 --no-sweep --no-cpu-baseline --no-online --no-e2e --batched-leg 0 --no-companion > gpurun_out/r50_$n.json 2>/dev/null
  timeout 900 python bench.py --net squeezenet1_0 --steps 30 --no-sweep --no-cpu-baseline --no-online --no-e2e --batched-leg 0 --no-companion > gpurun_out/sq10_$n.json 2>/dev/null
done
cp /tmp/libsecn_default.so paper_2506_11586_b200/libsecn.so
