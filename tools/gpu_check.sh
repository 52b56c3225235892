#!/bin/bash
# One gpurun pass: GPU tests, smoke, bench (both workloads + reference arm), ncu launch list + full capture.
# usage (on the box): bash tools/gpu_check.sh [tag]
tag=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 600 python bench.py > gpurun_out/${tag}_bench_kaggle.json 2> gpurun_out/${tag}_bench_kaggle.err
timeout 600 python bench.py --workload tb --no-cpu-baseline > gpurun_out/${tag}_bench_tb.json 2> gpurun_out/${tag}_bench_tb.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
if [ "${NCU:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${tag}_kaggle_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_dedup|k_insert|k_gather|k_pool|k_scatter|k_bwd|k_apply' -c 14 -o gpurun_out/${tag}_kaggle_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
fi
tail -3 gpurun_out/${tag}_pytest.log
