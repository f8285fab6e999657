# ncu of the target verify attention at B=64 (config 2) and B=256 (config 3's
# batch): why the kernel reaches 78 % of HBM at B=64 and ~47 % at B=256.
K="--profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled"
mkdir -p gpurun_out/r02f
for B in 64 256; do
  timeout 900 ncu $K -k "regex:k_attn_w<.int.128" -s 8 -c 1 -o gpurun_out/r02f/t_attn_b$B python scripts/profile_round.py --n-req $B --warm-rounds 40 > gpurun_out/r02f/ncu_b$B.log 2>&1
done
ls -la gpurun_out/r02f/
