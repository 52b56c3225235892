# A/B: cluster dedup on direct vs hashed big-table sets (harness + bench with the base library), interleaved
mkdir -p gpurun_out
out=gpurun_out/${1:-ab2}.txt
[ -n "$3" ] && { timeout 900 python -m pytest tests -m gpu -x -q $3 > gpurun_out/${1:-ab2}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${1:-ab2}_pytest.log; }
for r in $(seq ${2:-2}); do
  for sets in direct hashed; do echo "harness $sets $(./tools/dedup_bench kaggle 50 zipf 1 $sets | head -2 | tr '\n' ' ')" >> $out; done
  for v in "EC_LIB_NAME=libembcomm_gpu_base.so" "EC_CLUSTER_SETS=direct" "X=hashed"; do
    for w in ${WORKLOADS:-kaggle kaggle_hbm}; do
      env $v timeout 300 python bench.py --workload $w --no-cpu-baseline --schedule-batches 0 2>/dev/null | python tools/abline.py "$v $w" >> $out
    done
  done
done
cat $out
