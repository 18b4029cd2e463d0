"""Per-instruction profile of one kernel in an ncu report (source page, SASS):
opcode mix weighted by executions, and the hottest stall sites.
python tools/sass_hot.py REP [kernel-substring]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
blocks, cur = [], None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = [ln]
        blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
want = sys.argv[2] if len(sys.argv) > 2 else ""
for b in blocks:
    if want not in b[0]:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(b[1:]))))
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in hdr}
    tot_inst = 0
    ops = collections.Counter()
    stalls = []
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        ex = int(r[ix["Instructions Executed"]] or 0)
        samp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        ops[op] += ex
        tot_inst += ex
        stalls.append((samp, ex, r[ix["Address"]][-5:], src[:70],
                       {k: r[ix[k]] for k in ("stall_long_sb", "stall_wait", "stall_short_sb",
                                              "stall_math", "stall_lg", "stall_mio",
                                              "stall_branch_resolving", "stall_no_inst")}))
    print(b[0][:120])
    print("total warp instructions", tot_inst)
    for op, c in ops.most_common(25):
        print(f"  {op:10s} {c:12d} {100.0 * c / tot_inst:5.1f}%")
    tot_s = sum(s[0] for s in stalls)
    print("top stall sites (samples, execs):", tot_s)
    for s in sorted(stalls, reverse=True)[:30]:
        nz = {k: v for k, v in s[4].items() if v not in ("0", "")}
        print(f"  {s[0]:6d} {100.0*s[0]/max(tot_s,1):5.1f}% {s[1]:10d} {s[2]} {s[3]:70s} {nz}")
    break
