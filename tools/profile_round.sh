#!/bin/bash
# Round profile artefacts (run on the GPU box):  tools/profile_round.sh <tag>
#  gpurun_out/<tag>_launches.csv : launch list of bench.py (B200_PROFILING.md recipe)
#  gpurun_out/<tag>_full.ncu-rep : --set full of every kernel of one multiview render
# then here:  python tools/ncu_summary.py gpurun_out/<tag>_launches.csv gpurun_out/<tag>_full.ncu-rep \
#                 profiles/<tag>_traffic.json > profiles/<tag>_ncu.md
set -e
cd "$(dirname "$0")/.."
tag=${1:-r1}
ncu --metrics gpu__time_duration.sum --clock-control none -s 120 -c 64 --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 3 --warmup 5 --no-cpu-baseline --sorted-k 0 --no-backward \
    > gpurun_out/${tag}_launches.log 2>&1
# second render of view 1: skip pack_scene + the 16 kernels + rays of the first render
ncu --set full --import-source on --clock-control none -s 18 -c 16 -o gpurun_out/${tag}_full \
    python tools/render_view.py 1 2 > gpurun_out/${tag}_full.log 2>&1
# the next-row kernels: "Ours (sorted)" blend (k = 16) and the backward (K6)
KBUF=16 ncu --set full --import-source on --clock-control none -k regex:blend_kbuf -s 1 -c 1 -o gpurun_out/${tag}_kbuf \
    python tools/render_view.py 1 2 > gpurun_out/${tag}_kbuf.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:backward_kernel -s 1 -c 1 -o gpurun_out/${tag}_bwd \
    python tools/backward_view.py 1 2 > gpurun_out/${tag}_bwd.log 2>&1
