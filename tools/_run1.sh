timeout 600 python -m pytest tests/test_ga_gpu.py tests/test_functional_gpu.py tests/test_wide_gpu.py -q -x 2>&1 | tail -2
timeout 300 python tools/ga_large.py 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ga_launches.csv python -c "
import sys; sys.path.insert(0,'.')
from paper_1809_11134_b200 import GaConfig, GaEngine
from paper_1809_11134_b200.fitness import TargetSpec
from paper_1809_11134_b200.synthetic import haar_target
e=GaEngine(GaConfig(5,64,1<<20,max_generations=100,target_fitness=1.0),TargetSpec('h',5,haar_target(5)),1); e.set_launch_mode('kernels'); e.steps(2)
" > gpurun_out/ga_ncu.log 2>&1; echo rc=$?
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/ga_launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
agg=collections.defaultdict(list)
for r in rows[1:]:
    v=float(r[vi].replace(',','')); u=r[ui]
    v = v/1000 if u=='ns' else (v*1000 if u=='ms' else v)
    agg[r[ki][:70]].append(v)
for k,v in agg.items(): print(f"{k:70s} n={len(v)} mean_us={sum(v)/len(v):.1f}")
PY
