#!/bin/bash
# Full GPU evidence pass: tests, smoke, bench (ours, C4, reference arm), kernel
# sweeps, acceptance distributions, ncu launch list + full captures.
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --config c4 --steps 50 --warmup 5 --skip-cpu > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
ISQ_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 2 --warmup 3 --skip-e2e > $OUT/bench_n2_shared.json 2> $OUT/bench_n2_shared.err
timeout 600 python tools/kbench.py > $OUT/kbench.json 2>&1
timeout 300 python tools/small_bench.py > $OUT/small_bench.txt 2>&1
timeout 900 python tools/acceptance.py > $OUT/acceptance.json 2> $OUT/acceptance.err
timeout 300 python tools/ga_large.py > $OUT/ga_large.txt 2>&1
[ -x tools/susbench.bin ] && { tools/susbench.bin 1048576; tools/susbench.bin 65536; } > $OUT/susbench.txt 2>&1
if [ "${PROFILE:-1}" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $OUT/bench_launches.csv python bench.py --steps 2 --warmup 3 --skip-e2e --skip-fp32 --skip-extras > $OUT/bench_ncu.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fitness_fast|qeqea_values|qeqea_commit" -s 9 -c 3 \
      -o $OUT/prof_c5 python tools/engine_bench.py --P 1048576 --gens 2 > $OUT/ncu_full.log 2>&1
  echo "ncu rc=$?" >> $OUT/ncu_full.log
  for n in 3 4; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fitness_fast" -s 3 -c 1 \
      -o $OUT/prof_kb_n$n python tools/kbench.py --no-peak --prec fp64 --mix qeqea --only n$n --reps 2 > $OUT/ncu_n$n.log 2>&1
  done
fi
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; head -c 400 $OUT/bench.json; echo
