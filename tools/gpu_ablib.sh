# A/B of two library builds (libembcomm_gpu_base.so vs libembcomm_gpu.so) on bench workloads, interleaved
# usage: WORKLOADS="kaggle kaggle_hbm tb" bash tools/gpu_ablib.sh tag [rounds] [pytest-args]
tag=${1:-ablib}; mkdir -p gpurun_out; out=gpurun_out/${tag}.txt
[ -n "$3" ] && { timeout 900 python -m pytest tests -m gpu -x -q $3 > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log; }
for r in $(seq ${2:-2}); do
  for lib in libembcomm_gpu_base.so libembcomm_gpu.so; do
    for w in ${WORKLOADS:-kaggle kaggle_hbm}; do
      EC_LIB_NAME=$lib timeout 300 python bench.py --workload $w --no-cpu-baseline --schedule-batches 0 2>/dev/null | python tools/abline.py "$lib $w" >> $out
    done
  done
done
cat $out
