#!/bin/bash
# blend time vs GUT_BLEND_SEG (list entries per blend work item)
for s in 512 1024 2048 4096 16384 262144; do
  echo "SEG=$s"; GUT_BLEND_SEG=$s python tools/tile_work.py 1 2 3 2>&1 | grep -E "^view"
done
