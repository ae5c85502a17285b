#!/bin/bash
# race_check graph replays (trials 1, 3): e1 on the main branch with e3's branch empty, copying, or running e3
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for m in fork_empty fork_copy x; do
  for f in fire3 fire5 fire4 fire3; do
    echo "$m $f: $(timeout 200 python tools/race_check.py $f $m 2>&1 | grep 'full calls' | sed -E 's/.*trial ([0-9]) full calls \((eager|graph)\):/\1\2/' | grep -oE '^[0-9](eager|graph)|e[13]: out bad [0-9]+' | tr '\n' ' ')"
  done
done
