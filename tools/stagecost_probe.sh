# what a K2 stage costs the producer: traced per-stage cycles with the MMA removed (4), no slot
# back-pressure (4096), synthetic row indices (8192)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
rm -f gpurun_out/stagecost.log
for wl in C1 C2a; do
 for dbg in 0 4 4100 12292; do
  echo "=== $wl debug=$dbg" >> gpurun_out/stagecost.log
  TW_B200_DEBUG=$dbg timeout 120 python tools/trace_units.py --workload $wl --out-dtype fp16 --soak 2>&1 | grep -v Warn | grep -A8 "launch span\|producer cycles" | grep -v "^--" >> gpurun_out/stagecost.log
 done
done
cat gpurun_out/stagecost.log | grep -E "===|launch span|stage  [0-9]:|stage  1[01]:" 
