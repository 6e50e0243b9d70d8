set -u
OUT=gpurun_out
rm -f $OUT/kb_*.json
timeout 900 python -m pytest tests -m gpu -q -k "not c4" > $OUT/p1.log 2>&1; echo rc=$? >> $OUT/p1.log
for v in main nr4 nr16 multi4 old3; do
  lib=paper_1809_11134_b200/libisq.so; [ $v != main ] && lib=build/variants/$v/libisq.so
  ISQ_LIBRARY=$lib timeout 300 python tools/kbench.py --no-peak --prec fp64 --reps 40 > $OUT/kb_$v.json 2>&1
done
ISQ_LIBRARY=paper_1809_11134_b200/libisq.so timeout 300 python tools/kbench.py --no-peak --prec fp64 --reps 40 > $OUT/kb_main2.json 2>&1
timeout 300 python tools/kbench.py --no-peak --prec fp32 --reps 40 > $OUT/kb_fp32.json 2>&1
timeout 300 python tools/small_bench.py > $OUT/small.txt 2>&1
