# Round-2 evidence refresh after the attention / prefill changes (ev5_ files): GPU tests, bench
# lines (configs[1] default, reference arm, 13B scenario S, 72B, 7B scenario S), smoke, ncu launch
# list of one SD round, --set full of the 72B GQA attention + combine and of the 13B MHA attention.
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rs > gpurun_out/ev5_tests.log 2>&1
python bench.py > gpurun_out/ev5_n1.json 2> gpurun_out/ev5_n1.err
python bench.py --impl reference > gpurun_out/ev5_ref.json 2> gpurun_out/ev5_ref.err
python bench.py --workload cfg4 > gpurun_out/ev5_cfg4.json 2> gpurun_out/ev5_cfg4.err
python bench.py --workload cfg5 > gpurun_out/ev5_cfg5.json 2> gpurun_out/ev5_cfg5.err
python bench.py --workload s7b --no-attn-long --no-cpu-baseline > gpurun_out/ev5_s7b.json 2> gpurun_out/ev5_s7b.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev5_smoke.log 2>&1
python tools/attn_long.py > gpurun_out/ev5_attn_long.log 2>&1
python tools/prefill_time.py 7b 1024 64 > gpurun_out/ev5_prefill.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ev5_launches.csv python tools/prof_round.py > gpurun_out/ev5_ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"attn_gqa|attn_combine" --launch-skip 6 -c 2 \
    -o gpurun_out/ev5_gqa72b python tools/attn_long.py 72b > gpurun_out/ev5_ncu_g.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"attn_mha_tma|attn_combine" --launch-skip 6 -c 2 \
    -o gpurun_out/ev5_mha13b python tools/attn_long.py 13b > gpurun_out/ev5_ncu_m.log 2>&1
ls -la gpurun_out/ev5_*
