#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench lines, ncu launch list and
# one full ncu capture of the TW kernel.  Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,l2_cache_size --format=csv > gpurun_out/gpu.txt 2>&1 || true
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for wl in C2b C1 C5_75 C4; do timeout 600 python bench.py --workload $wl --no-cpu > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err; done
timeout 600 python bench.py --out-dtype fp32 --no-cpu > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err
TW_B200_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err
for wl in C2a C5_75 C2b C1; do timeout 300 python tools/ablate.py --workload $wl --debug 0 3 7 4 64; done > gpurun_out/ablate.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tw_gemm -s 3 -c 1 -o gpurun_out/prof_C2a -f python tools/ncu_step.py --workload C2a; timeout 900 ncu --set full --clock-control none --import-source on -k regex:tw_gemm -s 3 -c 1 -o gpurun_out/prof_C2a_fp16 -f python tools/ncu_step.py --workload C2a --out-dtype fp16; timeout 900 ncu --set full --clock-control none --import-source on -k regex:tw_gemm -s 3 -c 1 -o gpurun_out/prof_C5 -f python tools/ncu_step.py --workload C5_75 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:nvjet|gemm|cutlass" -s 6 -c 2 -o gpurun_out/prof_C2a_dense -f python tools/ncu_step.py --workload C2a --dense > gpurun_out/ncu_dense.log 2>&1
python tools/sass_hot.py gpurun_out/prof_C2a_fp16.ncu-rep 40 > gpurun_out/sass_hot_C2a_fp16.txt 2>&1
timeout 900 python tools/sweep.py --out gpurun_out/r01_sweep > gpurun_out/sweep.log 2>&1
ls -la gpurun_out
