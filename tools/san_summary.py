"""Summarise compute-sanitizer logs: errors grouped by kind and by the first
library / test host frames. Usage: python tools/san_summary.py LOG..."""
import collections
import re
import sys

for path in sys.argv[1:]:
    groups = collections.Counter()
    summary = []
    cur = None
    frames = []
    for line in open(path, errors="replace"):
        line = line.rstrip("\n")
        if "ERROR SUMMARY" in line or "RACECHECK SUMMARY" in line:
            summary.append(line.strip("= "))
            continue
        m = re.match(r"=========\s+(\S.*)", line)
        if not m:
            continue
        body = m.group(1)
        if body.startswith("Host Frame:") or body.startswith("Device Frame:"):
            f = re.sub(r"\[0x[0-9a-f]+\]", "", body.split(":", 1)[1]).strip()
            if ("libdyg" in f or ".py" in f or ".cu" in f) and len(frames) < 2:
                frames.append(f)
            continue
        if body.startswith(("Saved host", "Uninitialized access", "Access at", "at ")):
            continue
        if cur is not None:
            groups[(cur, tuple(frames))] += 1
        cur = re.sub(r"0x[0-9a-f]+", "ADDR", body)
        frames = []
    if cur is not None:
        groups[(cur, tuple(frames))] += 1
    print(f"== {path}")
    for s in summary:
        print("  " + s)
    for (kind, fr), n in groups.most_common(30):
        print(f"  {n:6d}  {kind}")
        for f in fr:
            print(f"          {f}")
