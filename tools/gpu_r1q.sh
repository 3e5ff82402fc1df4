timeout 300 python -m pytest tests/test_ops_gpu.py --timeout 120 -q -x 2>&1 | tail -2
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/q_bench.log 2>&1
tail -1 gpurun_out/q_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"
PB_RMSNORM_CTA=1 timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/q_bench_cta.log 2>&1
tail -1 gpurun_out/q_bench_cta.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cta', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"
timeout 300 python -m tests.step_breakdown 2 32 2>&1 | grep rmsnorm
