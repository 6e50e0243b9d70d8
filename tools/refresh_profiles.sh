#!/bin/bash
# Copy a tools/gpu_round.sh result (gpurun_out/) into the committed evidence
# under profiles/, named per round:   bash tools/refresh_profiles.sh r02
set -e
R=${1:-r02}
G=gpurun_out; P=profiles
cp $G/bench.json $P/${R}_bench_c5.json
cp $G/bench_c4.json $P/${R}_bench_c4.json
cp $G/bench_ref.json $P/${R}_bench_reference.json
cp $G/bench_n2_shared.json $P/${R}_bench_n2_shared_gpu_check.json
cp $G/kbench.json $P/${R}_kbench.json
cp $G/small_bench.txt $P/${R}_small_bench.txt
cp $G/acceptance.json $P/${R}_acceptance.json
grep -v "^==" $G/bench_launches.csv > $P/${R}_bench_launches.csv
python tools/summarize_ncu.py $G/prof_c5.ncu-rep $P/${R}_bench_launches.csv /tmp/${R}_c5 > /dev/null
cp /tmp/${R}_c5_ncu_full.json $P/${R}_c5_ncu_full.json
cp /tmp/${R}_c5_launches.md $P/${R}_c5_launches.md
python - "$R" <<'PY'
import json, sys
sys.path.insert(0, "tools")
from summarize_ncu import ncu_raw
r = sys.argv[1]
full = []
for n in (3, 4):
    full += ncu_raw(f"gpurun_out/prof_kb_n{n}.ncu-rep")
open(f"profiles/{r}_kb_n34_ncu_full.json", "w").write(json.dumps(full, indent=1))
PY
echo "refreshed profiles/${R}_*"
