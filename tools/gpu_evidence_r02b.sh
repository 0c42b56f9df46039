# Round-2 (late) evidence run: GPU tests, the driver's default bench twice, the reference arm,
# the full sweep over every BASELINE row, the bench launch list, ncu --set full of K2 at C2a
# (wide) and at C1 (narrow TB = 64 instantiation)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for i in 1 2; do
  timeout 900 python bench.py > gpurun_out/bench_default_$i.json 2> gpurun_out/bench_default_$i.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_default_$i.json')); print('default bench $i', round(d['ms_per_step']*1e3,2), 'us', round(d['speedup_vs_cublas_bf16'],2), 'x', d['clocks'], 'e2e', round(d['e2e']['ms_per_step'],3), 'ms')" || tail -3 gpurun_out/bench_default_$i.err
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_ref.json
timeout 1500 python tools/sweep.py --out gpurun_out/r02b_sweep > gpurun_out/sweep.log 2>&1; tail -3 gpurun_out/sweep.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-scale-point > /dev/null 2>&1; wc -l gpurun_out/launches_bench.csv
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tw_gemm -s 2 -c 1 -o gpurun_out/prof_r02b_C2a_K2 -f python tools/ncu_step.py --workload C2a --out-dtype fp16 --launches 3 > gpurun_out/ncu_C2a.log 2>&1; tail -1 gpurun_out/ncu_C2a.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tw_gemm -s 2 -c 1 -o gpurun_out/prof_r02b_C1_K2n -f python tools/ncu_step.py --workload C1 --out-dtype fp16 --launches 3 > gpurun_out/ncu_C1.log 2>&1; tail -1 gpurun_out/ncu_C1.log
