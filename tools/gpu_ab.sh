# interleaved A/B of environment variants on bench workloads (experiments); one summary line per run (tools/abline.py)
# usage: VARIANTS="X=0 EC_FOO=1,EC_BAR=2 EC_LIB_NAME=libembcomm_gpu_base.so" WORKLOADS="kaggle kaggle_hbm" bash tools/gpu_ab.sh tag [rounds] [pytest-args]
mkdir -p gpurun_out
tag=${1:-ab}; out=gpurun_out/${tag}.txt
[ -n "$3" ] && { timeout 900 python -m pytest tests -m gpu -x -q $3 > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log; }
for r in $(seq ${2:-2}); do
for v in ${VARIANTS:-"X=0"}; do
for w in ${WORKLOADS:-kaggle kaggle_hbm}; do
env ${v//,/ } timeout 300 python bench.py --workload $w --no-cpu-baseline --schedule-batches 0 2>/dev/null | python tools/abline.py "$v $w" >> $out
done; done; done
cat $out
