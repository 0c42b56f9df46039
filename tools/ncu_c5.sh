python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tw_gemm -s 2 -c 1 -o gpurun_out/prof_C5 -f python tools/ncu_step.py --workload C5_75 --launches 3 > gpurun_out/ncu_c5.log 2>&1
