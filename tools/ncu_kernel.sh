#!/bin/bash
# Source-level ncu capture of one kernel of a multiview render (GPU box):
#   tools/ncu_kernel.sh <kernel regex> <name> [launch skip] [view]
# then here:  python tools/sass_lines.py /tmp/<name>_sass.csv <nvdisasm sass> <mangled> <file>
set -e
cd "$(dirname "$0")/.."
ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${3:-0} -c 1 \
    -o gpurun_out/$2 python tools/render_view.py ${4:-1} 2 > gpurun_out/$2.log 2>&1
