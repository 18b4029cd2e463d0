#!/bin/bash
# GPU parity, then one C5 bench line per environment setting.
# Usage: gpurun -- bash tools/ab.sh TAG "ENV=.. ENV2=.." "ENV=.." ...   ("-" = defaults)
TAG=$1; shift
mkdir -p gpurun_out
if [[ "$TAG" != nt* ]]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
fi
i=0
for v in "$@"; do
  i=$((i+1))
  [ "$v" = "-" ] && v=""
  env $v timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ab_${TAG}_$i.json 2>gpurun_out/ab_${TAG}_$i.err
  python - "$v" gpurun_out/ab_${TAG}_$i.json <<'PY'
import json,sys
try:
    d=json.load(open(sys.argv[2]))
    p=d["phases_ms_per_step"]; r=d["roofline"]
    print(f"[{sys.argv[1] or 'default'}] ms/step={d['ms_per_step']:.3f} dev={d['device_ms_per_step']:.3f} restore={d.get('restore_ms_per_step',0):.3f} value={d['value']/1e6:.1f}M e2e={d['e2e']['value']/1e6:.1f}M frac={r['frac']:.3f} " + " ".join(f"{k.split()[0]}={v:.3f}" for k,v in p.items()) + f" delcommit={d['commit_ms_per_step_deletion_batches']:.3f} rounds={d['commit_rounds_per_step']} tail={d['walk_tail_ms_per_step']}")
except Exception as e:
    print("run", sys.argv[1], "failed", e)
PY
done
