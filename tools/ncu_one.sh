# one full ncu capture of the TW kernel: WL (workload), TAG (file suffix)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tw_gemm -s 2 -c 1 -o gpurun_out/prof_${TAG:-x} -f python tools/ncu_step.py --workload ${WL:-C2a} --launches 3 > gpurun_out/ncu_${TAG:-x}.log 2>&1
tail -3 gpurun_out/ncu_${TAG:-x}.log
