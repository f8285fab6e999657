for c in 128 256 512; do
  SPECTRE_ATTN_CHUNK=$c timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/attn_c$c.csv python scripts/profile_round.py --variant ordinary --warm-rounds 160 > /dev/null 2>&1
done
ls gpurun_out/attn_c*
