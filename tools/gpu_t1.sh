mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q > gpurun_out/t1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t1_pytest.log
for m in cluster tiles; do
timeout 300 python bench.py --no-cpu-baseline --schedule-batches 0 --dedup-mode $m > gpurun_out/t1_kaggle_$m.json 2>gpurun_out/t1_kaggle_$m.err
timeout 300 python bench.py --workload tb --no-cpu-baseline --schedule-batches 0 --dedup-mode $m > gpurun_out/t1_tb_$m.json 2>gpurun_out/t1_tb_$m.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_dedup' -c 2 -o gpurun_out/t1_dedup python bench.py --steps 1 --warmup 3 --no-cpu-baseline --schedule-batches 0 > /dev/null 2>&1
tail -5 gpurun_out/t1_pytest.log
