#!/bin/bash
# GPU box: tests + bench of the current tree.  tools/gpu_check.sh <tag> [pytest -k expr]
cd "$(dirname "$0")/.."
tag=${1:-chk}
if [ -n "$2" ]; then
  python -m pytest tests -m gpu -q -k "$2" > gpurun_out/${tag}_gputest.log 2>&1
else
  python -m pytest tests -m gpu -q > gpurun_out/${tag}_gputest.log 2>&1
fi
tail -3 gpurun_out/${tag}_gputest.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_bench.log 2>&1
python - "$tag" <<'PY'
import json, sys
for l in open(f"gpurun_out/{sys.argv[1]}_bench.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("value", round(d["value"], 1), "single", round(d["single_stream"]["frames_per_s"], 1),
              "e2e", round(d["e2e"]["value"], 1), {k: round(v, 4) for k, v in d["ms_stage"].items()})
PY
