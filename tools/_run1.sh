set -u
OUT=gpurun_out
for v in main m4_8 m4_12 m4_9; do
  lib=paper_1809_11134_b200/libisq.so; [ $v != main ] && lib=build/variants/$v/libisq.so
  ISQ_LIBRARY=$lib timeout 300 python tools/kbench.py --no-peak --prec fp64 --only n4 --reps 30 > $OUT/kb_$v.json 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -k "fitness" > $OUT/p1.log 2>&1; echo rc=$? >> $OUT/p1.log
