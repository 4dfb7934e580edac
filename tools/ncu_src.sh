#!/bin/bash
# Source-level capture of one kernel of the second render of multiview view 1.
# On the GPU box:  tools/ncu_src.sh capture <kernel-regex> <name>
# here:            tools/ncu_src.sh report <name> <mangled-function> <file.cu>  (uses the current build's SASS)
set -e
cd "$(dirname "$0")/.."
if [ "$1" = capture ]; then
  ncu --set full --clock-control none --import-source on -k regex:"$2" -s 1 -c 1 \
      -o gpurun_out/$3 python tools/render_view.py 1 2 > gpurun_out/$3.log 2>&1
else
  ncu -i gpurun_out/$2.ncu-rep --page source --csv --print-source sass > /tmp/$2_sass.csv 2>/dev/null
  obj=paper_2412_12507_b200/build/${4%.cu}.o
  d=$(mktemp -d); (cd $d && cuobjdump -xelf all "$OLDPWD/$obj" > /dev/null && nvdisasm --print-line-info *.cubin > /tmp/$2_lines.sass)
  python /tmp/lines2.py $2 $3 $4 1 100000
fi
