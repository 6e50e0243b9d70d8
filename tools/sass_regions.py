"""Summarise an ncu SASS source page (csv) by instruction-count blocks:
python tools/sass_regions.py report.ncu-rep kernel_regex [per_unit]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
unit = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
hdr = rows[hi[0]]
data = [dict(zip(hdr, r)) for r in rows[hi[0] + 1:(hi[1] if len(hi) > 1 else None)] if len(r) == len(hdr)]
S = [int(d["Warp Stall Sampling (All Samples)"]) for d in data]
I = [int(d["Instructions Executed"]) for d in data]
tot, it = sum(S), sum(I)
print(f"instructions {it} ({it / unit:.1f} per unit), samples {tot}")
ops = collections.Counter()
for d, n in zip(data, I):
    s = d["Source"].strip()
    ops[(s.split()[1] if s.startswith("@") else s.split()[0])] += n
print("top opcodes:", ", ".join(f"{k} {v / unit:.0f}" for k, v in ops.most_common(14)))
blocks, cur = [], None
for i, d in enumerate(data):
    e = I[i]
    if cur and cur[1] == e:
        cur[2].append(d["Source"].strip()); cur[3] += S[i]
    else:
        cur = [i, e, [d["Source"].strip()], S[i]]; blocks.append(cur)
for b in sorted(blocks, key=lambda b: -b[3])[:30]:
    c = collections.Counter((s.split()[1] if s.startswith("@") else s.split()[0]) for s in b[2])
    print(f"@{b[0]:5d} exec {b[1] / unit:7.2f} n {len(b[2]):4d} inst {b[1] * len(b[2]) / unit:7.1f} "
          f"samp {100 * b[3] / tot:5.1f}%  {c.most_common(6)}")
