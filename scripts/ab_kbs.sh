# decode step A/B: k-block slots per ring barrier (1 = one barrier per 64-column k-block)
for k in 1 default 2 4 8; do
  if [ $k = default ]; then unset HC_RING_KBS; else export HC_RING_KBS=$k; fi
  echo "kbs=$k $(timeout 300 python scripts/decode_probe.py 2>&1 | tail -1)"
done
unset HC_RING_KBS
