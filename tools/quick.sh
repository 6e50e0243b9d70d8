#!/bin/bash
# Quick GPU iteration: parity tests, kernel + engine throughput, optional ncu of one kernel.
#   NCU_K=<regex> bash tools/quick.sh    (adds a --set full capture of that kernel)
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q -x ${TESTS:-} > $OUT/q_pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/q_pytest.log
timeout 300 python tools/kbench.py --no-peak > $OUT/q_kbench.json 2>&1
timeout 300 python tools/engine_bench.py --P 1048576 --gens 6 > $OUT/q_engine.log 2>&1
if [ -n "${NCU_K:-}" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -s ${NCU_S:-4} -c 1 \
      -o $OUT/q_prof python tools/engine_bench.py --P 1048576 --gens 2 > $OUT/q_ncu.log 2>&1
  echo "ncu rc=$?" >> $OUT/q_ncu.log
fi
tail -2 $OUT/q_pytest.log; cat $OUT/q_kbench.json; cat $OUT/q_engine.log
