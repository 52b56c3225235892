mkdir -p gpurun_out
tag=${1:-x}
for m in auto atomic; do
timeout 300 python bench.py --no-cpu-baseline --schedule-batches 0 --scatter-mode $m --no-prefetch > gpurun_out/${tag}_kaggle_np_$m.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launch_$m.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --schedule-batches 0 --scatter-mode $m > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_bwd_apply|k_pool1|k_dedup' -c 6 -o gpurun_out/${tag}_fused python bench.py --steps 1 --warmup 3 --no-cpu-baseline --schedule-batches 0 > /dev/null 2>&1
