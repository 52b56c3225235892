mkdir -p gpurun_out
tag=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
for pr in 0 -1; do
for w in kaggle kaggle_hbm; do
timeout 300 python bench.py --workload $w --no-cpu-baseline --schedule-batches 0 --stream-priority $pr > gpurun_out/${tag}_${w}_p$pr.json 2>gpurun_out/${tag}_${w}_p$pr.err
done; done
tail -2 gpurun_out/${tag}_pytest.log
