# Round-2 evidence pass (on the box): GPU tests, smoke, every bench workload
# (BASELINE configs[0..3] at one GPU, both Kaggle tiers, the reference arm),
# ncu launch lists + full captures of the Kaggle and TB steps, dedup traces.
# usage: bash tools/gpu_r02.sh tag [skip-tests]
tag=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${tag}_smi.txt 2>&1
if [ -z "$2" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
fi
timeout 600 python bench.py > gpurun_out/${tag}_kaggle_bench.json 2> gpurun_out/${tag}_kaggle_bench.err
for w in kaggle_hbm tb cfg1 skew_uniform skew_zipf0.8 skew_zipf1.05 skew_zipf1.2 skew_bagpipe; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/${tag}_${w}_bench.json 2> gpurun_out/${tag}_${w}_bench.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_reference_bench.json 2> gpurun_out/${tag}_reference_bench.err
for w in kaggle tb; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${tag}_${w}_launches.csv python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --schedule-batches 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_dedup|k_insert|k_compact|k_inverse|k_gather|k_pool|k_scatter|k_bwd|k_apply|k_g64|k_patch' -c 16 -o gpurun_out/${tag}_${w}_full python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --schedule-batches 0 > /dev/null 2>&1
done
./tools/dedup_bench kaggle 50 > gpurun_out/${tag}_dedup_trace_kaggle.txt 2>&1
./tools/dedup_bench tb 20 > gpurun_out/${tag}_dedup_trace_tb.txt 2>&1
tail -2 gpurun_out/${tag}_pytest.log
