"""One line per bench JSON: ms/step, the phase split and K1's roofline."""
import json
import sys

for p in sorted(sys.argv[1:]):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(p, "unreadable", e)
        continue
    ph = {k.split(" ")[0]: round(v, 3) for k, v in d.get("phases_ms_per_step", {}).items()}
    gaps = {k: round(v, 3) for k, v in d.get("gaps_ms_per_step", {}).items()}
    tails = {k: round(v, 3) for k, v in d.get("walk_tail_ms_per_step", {}).items()}
    rf = d.get("roofline", {})
    print(f"{p.split('/')[-1]:40s} {d['ms_per_step']:.3f} ms  e2e {d['e2e']['value'] / 1e6:.1f} M/s  "
          f"{ph} gaps {gaps} tails {tails} frac {rf.get('frac', 0):.3f} "
          f"bulk {rf.get('frac_bulk', 0):.3f} tail {rf.get('frac_tail', 0):.3f}")
