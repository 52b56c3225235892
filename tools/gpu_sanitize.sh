mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 600 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s1_memcheck_smoke.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s1_racecheck_smoke.txt 2>&1
timeout 1200 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "small_fixed or heavy_misses or relays or csr or every_width or pools_a_zero_row" > gpurun_out/s1_memcheck_tests.txt 2>&1
for f in gpurun_out/s1_*.txt; do tail -n 3 $f; done
