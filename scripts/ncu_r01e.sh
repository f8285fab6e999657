# ncu evidence after the multi-block-stage GEMM and vectorised RoPE changes (round 1)
P="python scripts/profile_round.py --variant ordinary --warm-rounds 160"
K="--profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled"
timeout 600 ncu $K -k 'regex:swapab<.int.2, .int.64, .int.0' -s 40 -c 1 -o gpurun_out/d_swiglu_ksub $P > /dev/null 2>&1
timeout 600 ncu $K -k 'regex:swapab<.int.2, .int.64, .int.0' -s 50 -c 1 -o gpurun_out/t_swiglu $P > /dev/null 2>&1
timeout 600 ncu $K -k 'regex:k_qkv_rope_kv4' -s 60 -c 1 -o gpurun_out/rope4 $P > /dev/null 2>&1
timeout 600 ncu $K -k 'regex:swapab<.int.0, .int.64, .int.0' -s 3 -c 2 -o gpurun_out/t_partial_128 $P > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/round_launches_r01e.csv $P > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
