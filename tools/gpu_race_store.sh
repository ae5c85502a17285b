#!/bin/bash
# race_check graph replays (trials 1, 3) under epilogue variants of k_mac
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for v in "SECN_MAC_PLAINST=1" "SECN_MAC_BULKWAIT=1" "SECN_NONE=1"; do
  for f in fire3 fire5 fire4 fire3; do
    echo "$v $f: $(env $v timeout 200 python tools/race_check.py $f x 2>&1 | grep 'full calls' | sed -E 's/.*trial ([0-9]) full calls \((eager|graph)\):/\1\2/' | grep -oE '^[0-9](eager|graph)|e[13]: out bad [0-9]+' | tr '\n' ' ')"
  done
done
