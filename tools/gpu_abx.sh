# A/B of a kernel change: harness binaries (tools/dedup_bench_base vs tools/dedup_bench) and the
# bench step with the base library (EC_LIB_NAME=libembcomm_gpu_base.so) vs the new one, interleaved.
# usage: bash tools/gpu_abx.sh tag [rounds] [pytest-args]
tag=${1:-abx}; rounds=${2:-2}
mkdir -p gpurun_out
out=gpurun_out/${tag}.txt
[ -n "$3" ] && { timeout 900 python -m pytest tests -m gpu -x -q $3 > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log; }
for r in $(seq $rounds); do
  for b in dedup_bench_base dedup_bench; do
    [ -x tools/$b ] && for w in ${HARNESS:-kaggle tb}; do echo "$b $w $(./tools/$b $w 50 | head -1)" >> $out; done
  done
  for lib in libembcomm_gpu_base.so libembcomm_gpu.so; do
    for w in ${WORKLOADS:-kaggle kaggle_hbm}; do
      EC_LIB_NAME=$lib timeout 300 python bench.py --workload $w --no-cpu-baseline --schedule-batches 0 2>/dev/null | python tools/abline.py "$lib $w" >> $out
    done
  done
done
cat $out
