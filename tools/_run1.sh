for cfg in "4 32 131072" "4 32 262144" "5 64 65536" "5 64 131072" "5 16 262144" "3 16 262144"; do set -- $cfg; timeout 120 python -c "
import sys; sys.path.insert(0,'.')
from paper_1809_11134_b200 import GaConfig, GaEngine
from paper_1809_11134_b200.fitness import TargetSpec
from paper_1809_11134_b200.synthetic import haar_target
for mode in ['kernels']:
  try:
    e=GaEngine(GaConfig($1,$2,$3,max_generations=100,target_fitness=1.0),TargetSpec('h',$1,haar_target($1)),1); e.set_launch_mode(mode); e.steps(2); print('$cfg', mode, 'ok')
  except Exception as ex: print('$cfg', mode, 'FAIL', ex)
" 2>&1 | tail -1; done
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -c "
import sys; sys.path.insert(0,'.')
from paper_1809_11134_b200 import GaConfig, GaEngine
from paper_1809_11134_b200.fitness import TargetSpec
from paper_1809_11134_b200.synthetic import haar_target
e=GaEngine(GaConfig(4,32,262144,max_generations=100,target_fitness=1.0),TargetSpec('h',4,haar_target(4)),1); e.set_launch_mode('kernels'); e.steps(1)
" 2>&1 | grep -v "^=========     Host Frame" | head -40
