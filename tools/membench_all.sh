for b in membench3 membench4 membench6 mmabench membench5; do echo "=== $b"; timeout 120 tools/bin/$b; done > gpurun_out/membench.log 2>&1
