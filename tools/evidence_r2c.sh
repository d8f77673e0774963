set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rs > gpurun_out/ev6_tests.log 2>&1
python bench.py > gpurun_out/ev6_n1.json 2> gpurun_out/ev6_n1.err
python bench.py --impl reference > gpurun_out/ev6_ref.json 2> gpurun_out/ev6_ref.err
python bench.py --workload cfg4 > gpurun_out/ev6_cfg4.json 2> gpurun_out/ev6_cfg4.err
python bench.py --workload cfg5 > gpurun_out/ev6_cfg5.json 2> gpurun_out/ev6_cfg5.err
python bench.py --workload s7b --no-attn-long --no-cpu-baseline > gpurun_out/ev6_s7b.json 2> gpurun_out/ev6_s7b.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev6_smoke.log 2>&1
