# ncu evidence for the warp-per-item attention kernels (round 1, final)
P="python scripts/profile_round.py --variant ordinary --warm-rounds 160"
K="--profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled"
timeout 600 ncu $K -k 'regex:k_attn_w<.int.128' -s 4 -c 1 -o gpurun_out/t_attn_w $P > /dev/null 2>&1
timeout 600 ncu $K -k 'regex:k_attn_w<.int.64' -s 20 -c 1 -o gpurun_out/d_attn_w $P > /dev/null 2>&1
timeout 600 ncu $K -k 'regex:swapab<.int.0, .int.64, .int.1' -s 60 -c 3 -o gpurun_out/d_partial_half $P > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/round_launches_r01d.csv $P > /dev/null 2>&1
ls gpurun_out/*_w.ncu-rep gpurun_out/d_partial_half.ncu-rep
