# interleaved A/B of environment variants on bench workloads (experiments)
# usage: VARIANTS="X=0 EC_FOO=1,EC_BAR=2" WORKLOADS="kaggle kaggle_hbm" bash tools/gpu_ab.sh tag [rounds]
mkdir -p gpurun_out
out=gpurun_out/${1:-ab}.txt
for r in $(seq ${2:-2}); do
for v in ${VARIANTS:-"X=0"}; do
for w in ${WORKLOADS:-kaggle kaggle_hbm}; do
env ${v//,/ } timeout 300 python bench.py --workload $w --no-cpu-baseline --schedule-batches 0 2>/dev/null | sed "s/^/$v $w /" >> $out
done; done; done
