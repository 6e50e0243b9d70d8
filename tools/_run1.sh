set -u
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "functional or targets or resume" > $OUT/p1.log 2>&1; echo rc=$? >> $OUT/p1.log
timeout 900 python -m pytest tests -m gpu -q -k "not c4 and not functional and not targets and not resume" > $OUT/p2.log 2>&1; echo rc=$? >> $OUT/p2.log
