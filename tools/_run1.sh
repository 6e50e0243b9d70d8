set -u
OUT=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "not outcome_distributions" > $OUT/p1.log 2>&1; echo rc=$? >> $OUT/p1.log
timeout 300 python tools/kbench.py --no-peak --prec fp64 --reps 20 > $OUT/kb_main.json 2>&1
timeout 300 python tools/small_bench.py > $OUT/small_main.txt 2>&1
