# per-kernel context timings + full ncu captures of the top kernels (one ordinary round at ctx ~ 650)
set -x
timeout 400 python scripts/kprof.py --variant ordinary --warm-rounds 160 --rounds 3 > gpurun_out/kprof_ord.txt 2>&1
#timeout 400 python scripts/kprof.py --variant parallel --warm-rounds 200 --rounds 3 --out gpurun_out/kprof_par.json > gpurun_out/kprof_par.txt 2>&1
P="python scripts/profile_round.py --variant ordinary --warm-rounds 160"
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:swapab<.int.2' -s 48 -c 1 -o gpurun_out/gemm_gu_t $P > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_attention<.int.128' -c 1 -o gpurun_out/attn_t $P > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_attention<.int.64' -s 1 -c 1 -o gpurun_out/attn_d $P > gpurun_out/ncu3.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:swapab<.int.0' -s 4 -c 4 -o gpurun_out/gemm_d $P > gpurun_out/ncu4.log 2>&1
ls -la gpurun_out
