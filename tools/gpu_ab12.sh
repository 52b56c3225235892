mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab12_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab12_pytest.log
for b in dedup_bench_base dedup_bench; do echo "$b $(./tools/$b kaggle 50 | head -2 | tr '\n' ' ')" >> gpurun_out/ab12.txt; done
for lib in libembcomm_gpu_base.so libembcomm_gpu.so; do
  EC_LIB_NAME=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_dedup_cluster -c 4 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --schedule-batches 0 > gpurun_out/ab12_ncu_$lib.csv 2>/dev/null
  EC_LIB_NAME=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_dedup_cluster -c 4 --csv python bench.py --workload kaggle_hbm --steps 1 --warmup 3 --no-cpu-baseline --schedule-batches 0 > gpurun_out/ab12_ncuhbm_$lib.csv 2>/dev/null
done
