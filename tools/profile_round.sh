#!/bin/bash
# Capture the round's profiling evidence on a GPU box (run under gpurun):
#   1. plain run (must exit 0 before ncu touches it)
#   2. ncu launch list of 2 C4 frames (per-launch device time; shares, not absolutes)
#   3. ncu --set full of the top kernels at C4 (one launch each)
# Outputs land in gpurun_out/; tools/ncu_summary.py + tools/launch_shares.py
# turn them into profiles/.
set -e
OUT=gpurun_out
CMD="python tools/run_frames.py --config c4 --frames 3"
$CMD > $OUT/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_c4.csv $CMD > $OUT/ncu_launch.log 2>&1 || true
ncu --set full --clock-control none --import-source on \
    -k regex:"trace_kernel|blend_kernel|shadow_map|pack_delta|detect_kernel|build_kernel" \
    -s 9 -c 9 -o $OUT/full_c4 $CMD > $OUT/ncu_full.log 2>&1 || true
tail -2 $OUT/ncu_full.log
