set -u
OUT=gpurun_out
for n in 3 4 5; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fitness_fast" -s 3 -c 1 \
    -o $OUT/kb_n${n}_qeqea python tools/kbench.py --no-peak --prec fp64 --mix qeqea --only n$n --reps 2 > $OUT/ncu_n$n.log 2>&1
done
