#!/bin/bash
# race_check (fire e1/e3 on two streams, whole calls; trials 1 and 3 are graph replays) with and
# without programmatic dependent launch
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for v in 1 0; do
  for f in fire3 fire5 fire3 fire5 fire4; do
    echo "NO_PDL=$v $f: $(SECN_NO_PDL=$v timeout 200 python tools/race_check.py $f x 2>&1 | grep 'full calls' | sed -E 's/.*trial ([0-9]) full calls \((eager|graph)\):/\1\2/' | grep -oE '^[0-9](eager|graph)|e[13]: out bad [0-9]+' | tr '\n' ' ')"
  done
done
