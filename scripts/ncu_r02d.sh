# ncu evidence for the large-T verify GEMMs added late in round 2: the C3
# gate/up CTA pairs in 256-token chunks (T=1024) and the C5 (Qwen2.5-32B)
# 128-row gate/up at T=896 (one launch each, --set full).
K="--set full --import-source on --clock-control none --kernel-name-base demangled"
mkdir -p gpurun_out/r02d
timeout 900 ncu $K -k 'regex:swapab' -s 2 -c 1 -o gpurun_out/r02d/c3_gate_up_T1024 python scripts/one_gemm.py 28672 4096 2 1024 4000 > gpurun_out/r02d/ncu1.log 2>&1
timeout 900 ncu $K -k 'regex:swapab' -s 2 -c 1 -o gpurun_out/r02d/c5_gate_up_T896 python scripts/one_gemm.py 55296 5120 2 896 1000 > gpurun_out/r02d/ncu2.log 2>&1
ls -la gpurun_out/r02d/
