# Final bench lines of round 2 (ev8_ files): configs[1] default, 13B, 72B, 7B scenario S, reference arm
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/ev8_n1.json 2> gpurun_out/ev8_n1.err
python bench.py --workload cfg4 > gpurun_out/ev8_cfg4.json 2> gpurun_out/ev8_cfg4.err
python bench.py --workload cfg5 > gpurun_out/ev8_cfg5.json 2> gpurun_out/ev8_cfg5.err
python bench.py --workload s7b --no-attn-long --no-cpu-baseline > gpurun_out/ev8_s7b.json 2> gpurun_out/ev8_s7b.err
python bench.py --impl reference > gpurun_out/ev8_ref.json 2> gpurun_out/ev8_ref.err
python tools/attn_long.py > gpurun_out/ev8_attn_long.log 2>&1
python tools/prefill_time.py 7b 1024 64 > gpurun_out/ev8_prefill.log 2>&1
