# ncu evidence after the 64-token chain passes / register-store epilogues: the
# draft chains (a mid and the last chain of a 64-token decode step: launches
# 21 and 34 of the profiled round) and the launch list of one ordinary C2 round.
P="python scripts/profile_round.py --variant ordinary --warm-rounds 160"
K="--profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled"
mkdir -p gpurun_out/r02e
timeout 900 ncu $K -k "regex:k_chain" -s 20 -c 1 -o gpurun_out/r02e/d_chain_mid $P > gpurun_out/r02e/ncu1.log 2>&1
timeout 900 ncu $K -k "regex:k_chain" -s 33 -c 1 -o gpurun_out/r02e/d_chain_last $P > gpurun_out/r02e/ncu2.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e/round_launches_r02e.csv $P > gpurun_out/r02e/ncu3.log 2>&1
ls -la gpurun_out/r02e/
