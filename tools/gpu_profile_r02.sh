# Round-2 evidence run: GPU tests, the driver's default bench twice, ncu
# --set full captures of K2 (C2a) and K4 (C5 @ 0 %), the bench launch list,
# steady-state DRAM traffic of the K4 workloads.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do
  timeout 900 python bench.py > gpurun_out/bench_default_$i.json 2> gpurun_out/bench_default_$i.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_default_$i.json')); print('default bench $i', round(d['ms_per_step']*1e3,2), 'us', round(d['speedup_vs_cublas_bf16'],2), 'x', d['clocks'], 'e2e', round(d['e2e']['ms_per_step'],3), 'ms')" || tail -3 gpurun_out/bench_default_$i.err
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 400 gpurun_out/bench_ref.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tw_gemm -s 2 -c 1 -o gpurun_out/prof_r02_C2a_K2 -f python tools/ncu_step.py --workload C2a --out-dtype fp16 --launches 3 > gpurun_out/ncu_C2a.log 2>&1; tail -1 gpurun_out/ncu_C2a.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tw_pair -s 2 -c 1 -o gpurun_out/prof_r02_C5_0_K4 -f python tools/ncu_step.py --workload C5_0 --out-dtype fp16 --launches 3 > gpurun_out/ncu_C5_0.log 2>&1; tail -1 gpurun_out/ncu_C5_0.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-scale-point > /dev/null 2>&1; wc -l gpurun_out/launches_bench.csv
for spec in C5_0:fp16 C4:fp16; do
  wl=${spec%:*}; dt=${spec#*:}
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none \
    --clock-control none -k regex:tw_ -s 20 -c 40 --csv --log-file gpurun_out/traffic_${wl}_${dt}.csv \
    python tools/ncu_traffic.py run --workload $wl --out-dtype $dt > gpurun_out/traffic_${wl}_${dt}.log 2>&1
  tail -1 gpurun_out/traffic_${wl}_${dt}.log
done
