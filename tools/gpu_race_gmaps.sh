#!/bin/bash
# race_check (fire e1/e3 on two streams, whole calls) with the tensor maps in kernel parameters
# (default) and in per-CTA global copies (SECN_MAC_GMAPS=1)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for v in 0 1; do
  for f in fire3 fire5 fire3 fire5; do
    echo "GMAPS=$v $f: $(SECN_MAC_GMAPS=$v timeout 200 python tools/race_check.py $f x 2>&1 | grep 'full calls' | grep -oE 'e[13]: out bad [0-9]+' | tr '\n' ' ')"
  done
done
