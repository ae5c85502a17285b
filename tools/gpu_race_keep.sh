#!/bin/bash
# race_check graph replays under debug variants (comma-separated env settings per variant)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for v in ${VARIANTS:-SECN_TAIL_CV=1 SECN_TAIL_CV=1,SECN_NO_PDL=1}; do
  for f in fire3 fire5 fire4 fire3; do
    echo "$v $f: $(env $(echo $v | tr ',' ' ') timeout 200 python tools/race_check.py $f x 2>&1 | grep 'full calls' | sed -E 's/.*trial ([0-9]) full calls \((eager|graph)\):/\1\2/' | grep -oE '^[0-9](eager|graph)|e[13]: out bad [0-9]+' | tr '\n' ' ')"
  done
done
