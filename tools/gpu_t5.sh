mkdir -p gpurun_out
tag=${1:-x}
for args in "--dedup-mode tiles" "--dedup-mode cluster --scatter-mode transpose"; do
  n=$(echo $args | tr -d ' -')
  timeout 300 python bench.py --workload tb --no-cpu-baseline --schedule-batches 0 $args > gpurun_out/${tag}_tb_$n.json 2>/dev/null
  timeout 300 python bench.py --workload tb --no-cpu-baseline --schedule-batches 0 --no-prefetch $args > gpurun_out/${tag}_tbnp_$n.json 2>/dev/null
done
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --schedule-batches 0 > gpurun_out/${tag}_cfg1.json 2>/dev/null
./tools/dedup_bench tb 20 > gpurun_out/${tag}_db_tb.txt 2>&1
