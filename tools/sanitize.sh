#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the repo's kernels
# (mangled names under namespace ps) on config-1-sized work: smoke() (trace,
# tcgen05 blend, detect, assign, build, pack + delta), the codec / client /
# stream GPU tests.  Logs land in gpurun_out/san_*.log; run under gpurun.
cd "${GRAFT_REPO_ROOT:-.}"
OUT=gpurun_out
F="--kernel-name kns=_ZN2ps --print-limit 50 --error-exitcode 9"
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool $F python __graft_entry__.py smoke \
      > $OUT/san_${tool}_smoke.log 2>&1
  echo "smoke $tool exit $?" >> $OUT/san_summary.txt
done
timeout 1800 compute-sanitizer --tool memcheck $F python -m pytest -x -q \
    tests/test_gpu_codec.py tests/test_gpu_client.py tests/test_gpu_index.py \
    "tests/test_gpu_stream.py" -k "not full_size and not 131072" \
    > $OUT/san_memcheck_tests.log 2>&1
echo "tests memcheck exit $?" >> $OUT/san_summary.txt
timeout 900 compute-sanitizer --tool racecheck $F python -m pytest -x -q \
    tests/test_gpu_codec.py tests/test_gpu_index.py > $OUT/san_racecheck_tests.log 2>&1
echo "tests racecheck exit $?" >> $OUT/san_summary.txt
cat $OUT/san_summary.txt
for f in $OUT/san_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|========= (Invalid|Race|Barrier|Error)" $f | head -5; done
