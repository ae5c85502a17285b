#!/bin/bash
# C5 sweep (and a parity subset) under alternative builds of libsecn.so: every variants/*.so (built
# here with extra -D flags, git-ignored, shipped by gpurun) in turn replaces the in-tree library for
# one `bench.py --net ntt_sweep` run -> gpurun_out/sweep_<variant>.json; the default build is
# restored. VARIANT_ENV sets knobs for every run.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2506_11586_b200/libsecn.so /tmp/libsecn_default.so
for v in variants/*.so; do
  n=$(basename $v .so)
  cp $v paper_2506_11586_b200/libsecn.so; touch paper_2506_11586_b200/libsecn.so
  timeout 600 env ${VARIANT_ENV:-} python -m pytest tests/test_gpu_parity.py -q -x -k "ntt" > gpurun_out/pt_$n.log 2>&1
  timeout 600 env ${VARIANT_ENV:-} python bench.py --net ntt_sweep --steps 10 > gpurun_out/sweep_$n.json 2> gpurun_out/sweep_$n.err
done
cp /tmp/libsecn_default.so paper_2506_11586_b200/libsecn.so
