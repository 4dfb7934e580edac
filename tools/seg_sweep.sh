#!/bin/bash
# blend time vs GUT_BLEND_SEG (list entries per segment) x GUT_BLEND_WINDOW (segments in flight per unit)
for s in ${SEGS:-1024 2048 3072}; do
  for w in ${WINDOWS:-1 2 3}; do
    echo "SEG=$s WINDOW=$w"; GUT_BLEND_SEG=$s GUT_BLEND_WINDOW=$w timeout 120 python tools/tile_work.py 0 1 2 3 4 5 2>&1 | grep -E "^view"
  done
done
