# Round-1 evidence (run under gpurun, one GPU): bench line, ncu launch list of
# one SD round, one ncu --set full capture per kernel class, GQA attention.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r1b.csv python tools/prof_round.py > gpurun_out/ncu_l.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"gemm|attn" -c 6 -o gpurun_out/prof_r1b python tools/prof_round.py > gpurun_out/ncu_f.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"attn_gqa_tc" -c 1 \
    -o gpurun_out/prof_gqa python tools/attn_long.py 72b > gpurun_out/ncu_g.log 2>&1
