#!/bin/bash
# Capture the round's profiling evidence on a GPU box (run under gpurun), one
# ncu pass per gpurun call, each after the same command exited 0 without ncu:
#   tools/profile_round.sh launches  -> ncu launch list of 3 C4 frames
#                                       (per-launch device time; shares, not absolutes)
#   tools/profile_round.sh full      -> ncu --set full of the top kernels of frame 2
# Outputs land in gpurun_out/; tools/ncu_summary.py + tools/launch_shares.py
# turn them into profiles/.
set -e
OUT=gpurun_out
CMD="python tools/run_frames.py --config c4 --frames 3"
$CMD > $OUT/plain.log 2>&1
case "${1:-launches}" in
launches)
    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $OUT/launches_c4.csv $CMD > $OUT/ncu_launch.log 2>&1 || true
    tail -2 $OUT/ncu_launch.log ;;
full)
    ncu --set full --clock-control none --import-source on \
        -k regex:"trace_kernel|blend|shadow_map|pack_delta|detect_kernel|build_kernel|build_multi|bind_kernel|entries_kernel" \
        -s 13 -c 13 -o $OUT/full_c4 $CMD > $OUT/ncu_full.log 2>&1 || true
    tail -2 $OUT/ncu_full.log ;;
esac
