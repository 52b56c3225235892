mkdir -p gpurun_out
tag=${1:-x}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
for m in auto atomic; do
timeout 300 python bench.py --no-cpu-baseline --schedule-batches 0 --scatter-mode $m > gpurun_out/${tag}_kaggle_$m.json 2>gpurun_out/${tag}_kaggle_$m.err
timeout 300 python bench.py --workload kaggle_hbm --no-cpu-baseline --schedule-batches 0 --scatter-mode $m > gpurun_out/${tag}_kagglehbm_$m.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launch_$m.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --schedule-batches 0 --scatter-mode $m > /dev/null 2>&1
done
tail -3 gpurun_out/${tag}_pytest.log
