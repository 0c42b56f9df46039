# the N > 1 bench path (self-spawned ranks, gloo on one GPU: exercises the harness, timings not meaningful)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
TW_B200_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err
echo "rc=$?"; tail -c 1200 gpurun_out/bench_2rank_gloo.json; tail -5 gpurun_out/bench_2rank_gloo.err
