set -x
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/round_launches3.csv python scripts/profile_round.py --variant ordinary > gpurun_out/prof3.log 2>&1
timeout 400 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_attention -c 2 -o gpurun_out/attn python scripts/profile_round.py --variant ordinary > gpurun_out/prof_attn.log 2>&1
timeout 400 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gemm_bf16_swapab -c 6 -o gpurun_out/gemm python scripts/profile_round.py --variant ordinary > gpurun_out/prof_gemm.log 2>&1
ls -la gpurun_out
