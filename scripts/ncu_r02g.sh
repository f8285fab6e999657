# ncu of the target verify attention after the 7-warp / 2-stage change (B=256).
K="--profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled"
mkdir -p gpurun_out/r02g
timeout 900 ncu $K -k "regex:k_attn_w<.int.128" -s 8 -c 1 -o gpurun_out/r02g/t_attn7_b256 python scripts/profile_round.py --n-req 256 --warm-rounds 40 > gpurun_out/r02g/ncu.log 2>&1
ls -la gpurun_out/r02g/
