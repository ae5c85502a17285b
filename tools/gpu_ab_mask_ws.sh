python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for net in squeezenet1_1 resnet50; do
 for mask in host device; do
  for ws in 0 1; do
   SECN_MAC_WS=$ws timeout 900 python bench.py --net $net --mask $mask --no-sweep --no-cpu-baseline --no-companion --no-online --no-e2e --steps 20 > gpurun_out/ab_${net}_${mask}_ws$ws.json 2>&1
  done
 done
done
echo done
