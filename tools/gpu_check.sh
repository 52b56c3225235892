#!/bin/bash
# One gpurun pass: GPU tests, smoke, dedup harness, bench (kaggle + tb + reference arm), ncu launch list + full capture.
# usage (on the box): bash tools/gpu_check.sh [tag]
tag=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
[ -x tools/dedup_bench ] && { ./tools/dedup_bench kaggle 50 > gpurun_out/${tag}_db_kaggle.txt 2>&1; ./tools/dedup_bench tb 20 > gpurun_out/${tag}_db_tb.txt 2>&1; }
timeout 600 python bench.py > gpurun_out/${tag}_bench_kaggle.json 2> gpurun_out/${tag}_bench_kaggle.err
timeout 600 python bench.py --workload kaggle_hbm --no-cpu-baseline > gpurun_out/${tag}_bench_kagglehbm.json 2> gpurun_out/${tag}_bench_kagglehbm.err
timeout 600 python bench.py --workload tb --no-cpu-baseline > gpurun_out/${tag}_bench_tb.json 2> gpurun_out/${tag}_bench_tb.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
if [ "${NCU:-1}" = 1 ]; then
for w in kaggle tb; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${tag}_${w}_launches.csv python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --schedule-batches 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_dedup|k_insert|k_compact|k_inverse|k_gather|k_pool|k_scatter|k_bwd|k_apply|k_patch' -c 16 -o gpurun_out/${tag}_${w}_full python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --schedule-batches 0 > /dev/null 2>&1
done
fi
tail -3 gpurun_out/${tag}_pytest.log
