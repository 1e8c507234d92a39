set -x
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/c38_gpu_tests.txt 2>&1
tail -5 gpurun_out/c38_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c38_smoke.txt 2>&1
tail -3 gpurun_out/c38_smoke.txt
