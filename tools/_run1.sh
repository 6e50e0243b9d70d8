set -u
OUT=gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?" >> $OUT/bench.err
timeout 600 python bench.py --config c4 --steps 20 --warmup 3 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
