# ncu evidence, round 2 (final code): the draft chain, the verify gate/up, target split-K / attention, and the launch list of one ordinary round.
P="python scripts/profile_round.py --variant ordinary --warm-rounds 160"
K="--profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled"
mkdir -p gpurun_out/r02c
timeout 900 ncu $K -k 'regex:k_chain' -s 5 -c 1 -o gpurun_out/r02c/d_chain_mid $P > gpurun_out/r02c/ncu1.log 2>&1
timeout 900 ncu $K -k 'regex:k_chain' -s 16 -c 1 -o gpurun_out/r02c/d_chain_last $P > gpurun_out/r02c/ncu2.log 2>&1
timeout 900 ncu $K -k 'regex:swapab<.int.2, .int.64, .int.0, .int.1' -s 2 -c 1 -o gpurun_out/r02c/t_gate_up_pair $P > gpurun_out/r02c/ncu3.log 2>&1
timeout 900 ncu $K -k 'regex:swapab<.int.0, .int.64, .int.0, .int.0' -s 3 -c 3 -o gpurun_out/r02c/t_partial $P > gpurun_out/r02c/ncu4.log 2>&1
timeout 900 ncu $K -k 'regex:k_attn_w' -s 20 -c 2 -o gpurun_out/r02c/attn $P > gpurun_out/r02c/ncu5.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c/round_launches_r02c.csv $P > gpurun_out/r02c/ncu6.log 2>&1
ls -la gpurun_out/r02c/
