#!/bin/bash
# K5 source-level profile.  On the GPU box: tools/k5_profile.sh capture <name> [view]
# here: tools/k5_profile.sh report <name>   (uses the current build's SASS)
set -e
cd "$(dirname "$0")/.."
if [ "$1" = capture ]; then
  ncu --set full --clock-control none --import-source on -k regex:blend_kernel -s 1 -c 1 \
      -o gpurun_out/$2 python tools/render_view.py ${3:-1} 2 > gpurun_out/$2.log 2>&1
else
  ncu -i gpurun_out/$2.ncu-rep --page source --csv --print-source sass > /tmp/$2_sass.csv 2>/dev/null
  d=$(mktemp -d); (cd $d && cuobjdump -xelf all "$OLDPWD/paper_2412_12507_b200/build/k5_blend.o" > /dev/null \
     && nvdisasm --print-line-info *.cubin > /tmp/$2_lines.sass)
  python tools/k5_regions.py /tmp/$2_sass.csv /tmp/$2_lines.sass
fi
