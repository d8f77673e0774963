# Round-2 evidence on one GPU (final build: ev3_ files): GPU tests, bench lines (configs[1] default, the
# reference arm, configs[3] 13B scenario S, configs[4] 72B, 7B scenario S),
# ncu launch list of one SD round, --set full captures of the GEMM / attention
# classes and of the long-context MHA attention (13B, 4K context).
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rs > gpurun_out/ev3_tests.log 2>&1
python bench.py > gpurun_out/ev3_n1.json 2> gpurun_out/ev3_n1.err
python bench.py --impl reference > gpurun_out/ev3_ref.json 2> gpurun_out/ev3_ref.err
python bench.py --workload cfg4 > gpurun_out/ev3_cfg4.json 2> gpurun_out/ev3_cfg4.err
python bench.py --workload cfg5 > gpurun_out/ev3_cfg5.json 2> gpurun_out/ev3_cfg5.err
python bench.py --workload s7b --no-attn-long --no-cpu-baseline > gpurun_out/ev3_s7b.json 2> gpurun_out/ev3_s7b.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev3_smoke.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ev3_launches.csv python tools/prof_round.py > gpurun_out/ev3_ncu_l.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"gemm|attn" -c 7 -o gpurun_out/ev3_full python tools/prof_round.py > gpurun_out/ev3_ncu_f.log 2>&1
ncu --profile-from-start off --set full --clock-control none \
    -k regex:"gemm_tc" --launch-skip 32 -c 1 -o gpurun_out/ev3_head python tools/prof_round.py > gpurun_out/ev3_ncu_h.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"attn_mha_tma" --launch-skip 3 -c 1 \
    -o gpurun_out/ev3_mha13b python tools/attn_long.py 13b > gpurun_out/ev3_ncu_m.log 2>&1
ls -la gpurun_out/ev3_*
