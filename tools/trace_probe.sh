mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for spec in "C2a" "C2a --m 512" "C2b" "C5_75"; do
  echo "=== $spec" >> gpurun_out/trace.log
  timeout 120 python tools/trace_units.py --workload $spec --out-dtype fp16 --soak --cold >> gpurun_out/trace.log 2>&1
done
