# pair-dedup table size / retry rule (MST_DEDUP_TABLE_DIV, MST_DEDUP_RETRY)
mkdir -p gpurun_out
{
for c in ${CONFIGS:-c3 c2 c4}; do
  for v in "" MST_DEDUP_TABLE_DIV=2 MST_DEDUP_RETRY=1 "MST_DEDUP_TABLE_DIV=2 MST_DEDUP_RETRY=1" MST_DEDUP_TABLE_DIV=1; do
    echo -n "$c ${v:-base}: "; env $v timeout 300 python tools/mst_once.py --config $c --warmup 2 --reps 5 | head -2 | tr '\n' ' '; echo
  done
done
} > gpurun_out/sweep_dedup.log 2>&1
