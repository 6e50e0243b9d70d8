set -u
OUT=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "not outcome_distributions" > $OUT/p1.log 2>&1; echo rc=$? >> $OUT/p1.log
timeout 600 python bench.py --steps 20 --warmup 3 --skip-e2e --skip-fp32 --skip-extras > $OUT/b_main.json 2> $OUT/b_main.err
