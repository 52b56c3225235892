# HBM tier: prefetch depth 1 (default) vs 2, with and without row sources (interleaved rounds)
mkdir -p gpurun_out; out=gpurun_out/${1:-abd}.txt
for r in 1 2 3; do
 for w in kaggle_hbm skew_uniform; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --schedule-batches 0 2>/dev/null | python tools/abline.py "depth1 $w" >> $out
  timeout 300 python bench.py --workload $w --prefetch-depth 2 --no-cpu-baseline --schedule-batches 0 2>/dev/null | python tools/abline.py "depth2 $w" >> $out
  EC_ROW_SOURCES=all timeout 300 python bench.py --workload $w --prefetch-depth 2 --no-cpu-baseline --schedule-batches 0 2>/dev/null | python tools/abline.py "depth2+rsrc $w" >> $out
  EC_ROW_SOURCES=all EC_PF_DELAY_NS=0 timeout 300 python bench.py --workload $w --prefetch-depth 2 --no-cpu-baseline --schedule-batches 0 2>/dev/null | python tools/abline.py "depth2+rsrc+nodelay $w" >> $out
 done
done
cat $out
