# ncu --set full capture of the main kernel at one sweep point (used for profiles/).
set -x
SL=${1:-2048}
SCHED=${2:-shift}
TAG=${3:-r01}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dash_bwd_kernel -s 2 -c 1 \
  -o gpurun_out/prof_${TAG}_${SCHED}_n${SL} python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e \
  --seqlens ${SL} --schedule ${SCHED} > gpurun_out/ncu_full_${TAG}_${SCHED}_n${SL}.log 2>&1
tail -3 gpurun_out/ncu_full_${TAG}_${SCHED}_n${SL}.log
