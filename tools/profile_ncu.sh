# ncu evidence of the current build (one GPU): launch list of one SD round, one
# --set full capture per kernel class (first 6 GEMM/attention launches + the head GEMM)
mkdir -p gpurun_out
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r1e.csv python tools/prof_round.py > gpurun_out/ncu_l.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"gemm|attn" -c 6 -o gpurun_out/prof_r1e python tools/prof_round.py > gpurun_out/ncu_f.log 2>&1
ncu --profile-from-start off --set full --clock-control none \
    -k regex:"gemm_tc" --launch-skip 32 -c 1 -o gpurun_out/prof_head python tools/prof_round.py > gpurun_out/ncu_h.log 2>&1
