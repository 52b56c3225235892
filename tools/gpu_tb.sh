# TB / cfg1 iteration: engine GPU tests, TB + cfg1 + skew benches (usage: bash tools/gpu_tb.sh tag [extra bench args])
mkdir -p gpurun_out
tag=${1:-t}; shift
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
for w in tb cfg1 tb; do
timeout 300 python bench.py --workload $w --no-cpu-baseline --schedule-batches 0 "$@" >> gpurun_out/${tag}_${w}.json 2>>gpurun_out/${tag}_${w}.err
done
tail -2 gpurun_out/${tag}_pytest.log
