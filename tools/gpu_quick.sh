# quick loop: engine GPU tests + kaggle benches (usage: bash tools/gpu_quick.sh tag [extra bench args])
mkdir -p gpurun_out
tag=${1:-x}; shift
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python bench.py --no-cpu-baseline --schedule-batches 0 "$@" > gpurun_out/${tag}_kaggle.json 2>gpurun_out/${tag}_kaggle.err
timeout 300 python bench.py --no-cpu-baseline --schedule-batches 0 "$@" > gpurun_out/${tag}_kaggle2.json 2>/dev/null
timeout 300 python bench.py --workload kaggle_hbm --no-cpu-baseline --schedule-batches 0 "$@" > gpurun_out/${tag}_kagglehbm.json 2>/dev/null
tail -2 gpurun_out/${tag}_pytest.log
