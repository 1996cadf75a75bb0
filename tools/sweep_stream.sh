# streamed e2e path (tools/prof_stream.py): wall ms of 6 calls per setting, sorted
run() { echo "$1 $(env $1 python tools/prof_stream.py --reps 6 $2 2>&1 | grep packed | awk '{print $2}' | sort -n | tr '\n' ' ')"; }
run "DM_STREAM_RAW_MB=32 DM_STREAM_BIG_MB=128"
run "DM_STREAM_RAW_MB=16 DM_STREAM_BIG_MB=128"
run "DM_STREAM_RAW_MB=32 DM_STREAM_BIG_MB=64"
run "DM_STREAM_RAW_MB=16 DM_STREAM_BIG_MB=64"
run "DM_STREAM_RAW_MB=32 DM_STREAM_BIG_MB=128 DM_STREAM_RAW_FRAC=0.35"
run "DM_STREAM_RAW_MB=32 DM_STREAM_BIG_MB=128 DM_STREAM_RAW_FRAC=0.25"
run "DM_STREAM_RAW_MB=32 DM_STREAM_BIG_MB=128 DM_STREAM_SMALL_MB=16"
run "DM_STREAM_BIG_MB=128" --pageable
run "DM_STREAM_BIG_MB=64" --pageable
run "DM_STREAM_BIG_MB=256" --pageable
