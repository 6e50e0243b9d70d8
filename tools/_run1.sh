tools/susbench.bin 1048576 | tail -5; tools/susbench.bin 65536 | tail -5
timeout 600 python -m pytest tests/test_ga_gpu.py tests/test_functional_gpu.py -q -x 2>&1 | tail -2
ISQ_LIBRARY=build/variants/susprof/libisq.so timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1809_11134_b200 import GaConfig, GaEngine
from paper_1809_11134_b200.fitness import TargetSpec
from paper_1809_11134_b200.synthetic import haar_target
e=GaEngine(GaConfig(5,64,1<<20,max_generations=100,target_fitness=1.0),TargetSpec('h',5,haar_target(5)),1); e.set_launch_mode('kernels'); e.steps(2)
" 2>&1 | tail -4
timeout 300 python tools/ga_large.py 2>&1 | tail -1
