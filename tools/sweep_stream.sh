# streamed e2e path (tools/prof_stream.py): wall ms of 6 calls per setting, sorted
for hw in 16; do for f in 0.25 0.3 0.35 0.4; do
echo "hwsel=$hw frac=$f $(DM_STREAM_HWSEL=$hw DM_STREAM_RAW_FRAC=$f python tools/prof_stream.py --reps 6 2>&1 | grep packed | awk '{print $2}' | sort -n | tr '\n' ' ')"
done; done
echo "pageable $(python tools/prof_stream.py --reps 6 --pageable 2>&1 | grep packed | awk '{print $2}' | sort -n | tr '\n' ' ')"
