#!/bin/bash
# Round profile artefacts (run on the GPU box):  tools/profile_round.sh <tag>
#  gpurun_out/<tag>_launches.csv : launch list of bench.py (B200_PROFILING.md recipe)
#  gpurun_out/<tag>_full.ncu-rep : --set full of every kernel of one multiview render (the 2nd)
#  gpurun_out/<tag>_<config>.ncu-rep : --set full of K1 and K5 of one view of the other configs
#  gpurun_out/<tag>_kbuf / _bwd  : the next-row kernels ("Ours (sorted)" blend, backward)
# then here:  python tools/ncu_summary.py gpurun_out/<tag>_launches.csv gpurun_out/<tag>_full.ncu-rep \
#                 profiles/<tag>_traffic.json > profiles/<tag>_ncu.md
set -e
cd "$(dirname "$0")/.."
tag=${1:-r2}
part=${2:-all}   # main | configs | next | all  (gpurun brings back <= 64 MiB per call)
if [ "$part" = main ] || [ "$part" = all ]; then
# launch list of bench.py's timed region (NVTX range bench_timed)
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "bench_timed/" --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 4 --warmup 5 --no-cpu-baseline --sorted-k 0 --no-backward \
    > gpurun_out/${tag}_launches.log 2>&1
# second render of view 1: skip the scene pack + the first render (18 kernels + the ray table)
ncu --set full --clock-control none -s 18 -c 16 -o gpurun_out/${tag}_full \
    python tools/render_view.py 1 2 > gpurun_out/${tag}_full.log 2>&1
fi
if [ "$part" = configs ] || [ "$part" = all ]; then
for cfg in waymo mipnerf360 scannetpp; do
  TRACE_CONFIG=$cfg ncu --set full --clock-control none \
      -k regex:"project_prefilter|project_kernel|blend_kernel" -s 3 -c 3 -o gpurun_out/${tag}_${cfg} \
      python tools/render_view.py 1 2 > gpurun_out/${tag}_${cfg}.log 2>&1
done
fi
if [ "$part" = next ] || [ "$part" = all ]; then
# the next-row kernels: "Ours (sorted)" blend (k = 16) and the backward (K6)
KBUF=16 ncu --set full --clock-control none -k regex:blend_kbuf -s 1 -c 1 -o gpurun_out/${tag}_kbuf \
    python tools/render_view.py 1 2 > gpurun_out/${tag}_kbuf.log 2>&1
ncu --set full --clock-control none -k regex:backward_kernel -s 1 -c 1 -o gpurun_out/${tag}_bwd \
    python tools/backward_view.py 1 2 > gpurun_out/${tag}_bwd.log 2>&1
fi
