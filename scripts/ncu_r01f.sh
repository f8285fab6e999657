# ncu evidence for the CTA-pair (cta_group::2) target gate/up GEMM (round 1)
P="python scripts/profile_round.py --variant ordinary --warm-rounds 160"
K="--profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled"
timeout 600 ncu $K -k 'regex:swapab<.int.2, .int.64, .int.0, .int.1' -s 2 -c 1 -o gpurun_out/t_swiglu_pair $P > /dev/null 2>&1
ls -la gpurun_out/t_swiglu_pair.ncu-rep
