# ncu evidence for round 1 (one ordinary round at ctx ~650, C2 shapes)
set -x
P="python scripts/profile_round.py --variant ordinary --warm-rounds 160"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/round_launches_r01c.csv $P > /dev/null 2>&1
# draft step kernels come first in an ordinary round (3 steps x 16 layers), then the target (32 layers)
K="--profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled"
timeout 600 ncu $K -k 'regex:swapab<.int.2' -s 48 -c 1 -o gpurun_out/t_gate_up $P > /dev/null 2>&1
timeout 600 ncu $K -k 'regex:swapab<.int.0' -s 146 -c 3 -o gpurun_out/t_partial $P > /dev/null 2>&1
timeout 600 ncu $K -k 'regex:swapab<.int.2' -s 20 -c 1 -o gpurun_out/d_gate_up $P > /dev/null 2>&1
timeout 600 ncu $K -k 'regex:swapab<.int.0' -s 60 -c 3 -o gpurun_out/d_partial $P > /dev/null 2>&1
timeout 600 ncu $K -k 'regex:swapab<.int.1' -s 3 -c 1 -o gpurun_out/t_lm_head $P > /dev/null 2>&1
timeout 600 ncu $K -k 'regex:k_attn<.int.128' -s 4 -c 1 -o gpurun_out/t_attn $P > /dev/null 2>&1
timeout 600 ncu $K -k 'regex:k_attn<.int.64' -s 20 -c 1 -o gpurun_out/d_attn $P > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
