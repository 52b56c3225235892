mkdir -p gpurun_out
tag=${1:-x}
./tools/dedup_bench kaggle 50 > gpurun_out/${tag}_db_kaggle.txt 2>&1
./tools/dedup_bench tb 20 > gpurun_out/${tag}_db_tb.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python bench.py --no-cpu-baseline --schedule-batches 0 > gpurun_out/${tag}_kaggle.json 2>gpurun_out/${tag}_kaggle.err
timeout 300 python bench.py --workload tb --no-cpu-baseline --schedule-batches 0 > gpurun_out/${tag}_tb.json 2>gpurun_out/${tag}_tb.err
tail -3 gpurun_out/${tag}_pytest.log
