# dedup iteration: harness (both shapes, zipf/uniform, tag on/off), engine GPU tests, Kaggle benches
# usage (on the box): bash tools/gpu_dedup.sh tag [ncu]
tag=${1:-d}
mkdir -p gpurun_out
for w in kaggle tb; do for d in zipf uniform; do
  timeout 120 ./tools/dedup_bench $w 50 $d 1 > gpurun_out/${tag}_db_${w}_${d}.txt 2>&1
done; done
timeout 120 ./tools/dedup_bench kaggle 50 zipf 0 > gpurun_out/${tag}_db_kaggle_notag.txt 2>&1
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_engine.py -x -q -m gpu -k "every_width" >> gpurun_out/${tag}_width.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${tag}_kaggle.json 2>gpurun_out/${tag}_kaggle.err
timeout 300 python bench.py --workload kaggle_hbm --no-cpu-baseline > gpurun_out/${tag}_kagglehbm.json 2>/dev/null
if [ -n "$2" ]; then
timeout 300 ncu --set full --clock-control none -k regex:k_dedup_cluster -c 2 -o gpurun_out/${tag}_db_kaggle ./tools/dedup_bench kaggle 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_dedup_cluster -c 2 -o gpurun_out/${tag}_db_tb ./tools/dedup_bench tb 3 > /dev/null 2>&1
fi
tail -2 gpurun_out/${tag}_pytest.log
