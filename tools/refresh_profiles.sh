#!/bin/bash
# Copy a gpu_round.sh result (gpurun_out/) into the committed round-1 evidence under profiles/.
set -e
G=gpurun_out; P=profiles
cp $G/bench.json $P/r01_bench_c5.json
cp $G/bench_ref.json $P/r01_bench_reference.json
cp $G/kbench.json $P/r01_kbench.json
cp $G/small_bench.txt $P/r01_small_bench.txt
cp $G/acceptance.json $P/r01_acceptance.json
[ -s $G/rb.txt ] && cp $G/rb.txt $P/r01_randbench.txt
python tools/summarize_ncu.py $G/prof_c5.ncu-rep $G/launches_c5.csv /tmp/r01_c5 > /dev/null
cp /tmp/r01_c5_ncu_full.json $P/r01_c5_ncu_full.json
cp /tmp/r01_c5_launches.md $P/r01_c5_launches.md
grep -v "^==" $G/launches_c5.csv > $P/r01_launches_c5.csv
grep -v "^==" $G/bench_launches.csv > $P/r01_bench_launches.csv
python - <<'PY'
import csv, json
from collections import defaultdict
rows = list(csv.reader(open('profiles/r01_bench_launches.csv')))
h = rows[0]
ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per, order = defaultdict(list), []
for r in rows[1:]:
    if len(r) > iv and r[im] == "gpu__time_duration.sum":
        k = r[ik].split("(")[0].replace("void ", "")
        if k not in per:
            order.append(k)
        per[k].append(float(r[iv].replace(",", "")))
gen = {"fma_peak_kernel<double>", "qeqea_init_kernel"}
tot = sum(sum(per[k]) / len(per[k]) for k in order if k not in gen)
b = json.load(open('gpurun_out/bench.json'))
sc = b['phase_ms']['score (fitness kernel)']
ms = b['ms_per_step']
L = ["# ncu launch list of `python bench.py --steps 2 --warmup 3 --skip-e2e --skip-fp32`", "",
     "`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: compare shares).  "
     f"The fitness kernel's share agrees with the bench's phase timing (score = {sc:.2f} of {ms:.1f} ms, "
     f"{sc / ms:.0%} of a generation).", "",
     "| kernel | launches | mean (us) | share of a generation |", "|---|---|---|---|"]
for k in order:
    m = sum(per[k]) / len(per[k])
    L.append(f"| {k} | {len(per[k])} | {m / 1e3:.1f} | {'—' if k in gen else f'{m / tot:.1%}'} |")
open('profiles/r01_bench_launches.md', 'w').write("\n".join(L) + "\n")
PY
