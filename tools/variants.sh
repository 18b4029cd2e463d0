#!/bin/bash
# Walk-kernel variant sweep on C5: GPU parity first, then one bench line per variant.
# Usage: gpurun -- bash tools/variants.sh TAG "R M" "R M" ...   (R = DYG_WALK_REACH, M = DYG_WALK_MIN)
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
for v in "$@"; do
  set -- $v
  DYG_WALK_REACH=$1 DYG_WALK_MIN=$2 timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/var_${TAG}_$1_$2.json 2>/dev/null
  python - "$1" "$2" gpurun_out/var_${TAG}_$1_$2.json <<'PY'
import json,sys
try:
    d=json.load(open(sys.argv[3]))
    p=d["phases_ms_per_step"]; r=d["roofline"]
    print(f"reach={sys.argv[1]} min={sys.argv[2]} ms/step={d['ms_per_step']:.3f} value={d['value']/1e6:.1f}M e2e={d['e2e']['value']/1e6:.1f}M frac={r['frac']:.3f} " + " ".join(f"{k.split()[0]}={v:.3f}" for k,v in p.items()) + f" tail={d['walk_tail_ms_per_step']}")
except Exception as e:
    print("variant", sys.argv[1], sys.argv[2], "failed", e)
PY
done
