set -u
OUT=gpurun_out
rm -f $OUT/kb_*.json $OUT/small_*.txt
timeout 900 python -m pytest tests -m gpu -q -x -k "not c4" > $OUT/p1.log 2>&1; echo rc=$? >> $OUT/p1.log
timeout 300 python tools/kbench.py --no-peak --prec fp64 --reps 40 > $OUT/kb_main.json 2>&1
timeout 300 python tools/small_bench.py > $OUT/small_main.txt 2>&1
