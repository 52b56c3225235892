mkdir -p gpurun_out
for r in 1 2 3; do
for lib in libembcomm_gpu_prev.so libembcomm_gpu.so; do
for w in kaggle kaggle_hbm; do
EC_LIB_NAME=$lib timeout 300 python bench.py --workload $w --no-cpu-baseline --schedule-batches 0 | sed "s/^/$lib $w /" >> gpurun_out/ab1.txt 2>/dev/null
done; done; done
