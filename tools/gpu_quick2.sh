mkdir -p gpurun_out
tag=${1:-x}; shift
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
for w in kaggle kaggle_hbm tb cfg1; do
timeout 300 python bench.py --workload $w --no-cpu-baseline --schedule-batches 0 "$@" > gpurun_out/${tag}_$w.json 2>gpurun_out/${tag}_$w.err
done
timeout 300 python bench.py --workload tb --no-cpu-baseline --schedule-batches 0 --scatter-mode transpose > gpurun_out/${tag}_tb_old.json 2>/dev/null
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --schedule-batches 0 --scatter-mode transpose > gpurun_out/${tag}_cfg1_old.json 2>/dev/null
tail -2 gpurun_out/${tag}_pytest.log
