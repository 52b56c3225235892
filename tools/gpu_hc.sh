mkdir -p gpurun_out
tag=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
python tools/hostcost.py kaggle 300 > gpurun_out/${tag}_hc.txt 2>&1; python tools/hostcost.py kaggle_hbm 300 >> gpurun_out/${tag}_hc.txt 2>&1
for i in 1 2; do for w in kaggle kaggle_hbm; do
timeout 300 python bench.py --workload $w --no-cpu-baseline --schedule-batches 0 > gpurun_out/${tag}_${w}_$i.json 2>gpurun_out/${tag}_${w}_$i.err
done; done
tail -2 gpurun_out/${tag}_pytest.log
