timeout 300 python -m pytest tests/test_gemm_gpu.py --timeout 120 -q -x 2>&1 | tail -2
timeout 600 python -m pytest tests/test_executor_gpu.py --timeout 240 -q -x 2>&1 | tail -2
timeout 700 python bench.py > gpurun_out/p_bench.log 2>&1
tail -1 gpurun_out/p_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['mfu'], d['loss'], d['clocks'])"
