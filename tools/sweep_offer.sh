# offer-mode sweep per call site (MST_OFFER_<SITE> = 0 plain RED, 1 read-first, 2 read-first batched)
mkdir -p gpurun_out
{
for c in ${CONFIGS:-c1 c0 c2 c3 c4}; do
  for v in "" MST_OFFER_MIN1=0 MST_OFFER_MIN1=2 MST_OFFER_COUNT=0 MST_OFFER_COUNT=2 MST_OFFER_SPLIT=0 MST_OFFER_SPLIT=2 MST_OFFER_HEAVY=0 MST_OFFER_HEAVY=2; do
    echo -n "$c ${v:-base}: "; env $v timeout 300 python tools/mst_once.py --config $c --warmup 3 --reps ${REPS:-10} | head -1
  done
done
} > gpurun_out/sweep_offer.log 2>&1
