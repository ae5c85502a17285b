#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build_st.log 2>&1 || { echo build failed; tail -20 $O/build_st.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_st.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_st.log
for i in 1 2 3 4 5 6; do STAGED=1 timeout 200 python tools/online_check.py 2>&1 | grep mismatches | tr "\n" " "; echo; done
timeout 600 python bench.py > $O/bench_full_st.json 2> $O/bench_full_st.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$O/bench_full_st.json').read().strip().splitlines()[-1]);print('STEP_MS',d['ms_per_step'],d['roofline']['frac'],d['cpu_baseline'].get('parity_mismatched_words_on_sample'),d['clocks'])"
