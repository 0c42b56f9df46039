# per-unit timelines of one launch under experiment knobs (TW_B200_DEBUG bits:
# 1 skip zero rows, 2 skip kept-row stores, 4 skip MMA, 8 no proxy fence,
# 16 staging reads without global store, 32 zero rows by TMA bulk stores)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for wl in ${WLS:-C5_75 C2b C2a}; do
 for dbg in ${DBGS:-0 32 1 2 3 7}; do
  echo "=== $wl debug=$dbg" >> gpurun_out/trace.log
  TW_B200_DEBUG=$dbg timeout 120 python tools/trace_units.py --workload $wl ${TRACE_ARGS} >> gpurun_out/trace.log 2>&1
 done
done
