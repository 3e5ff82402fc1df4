timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_ops_gpu.py --timeout 120 -q 2>&1 | tail -3
timeout 900 python -m pytest tests/test_executor_gpu.py tests/test_multiprocess_gpu.py --timeout 240 -q 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/h_bench.log 2>&1
tail -1 gpurun_out/h_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['mfu'], d['clocks'], d['activation_memory']['pool_bytes_per_device'])"
timeout 1500 python tools/projection.py --model 1.5b --p 2 4 8 --balance --out gpurun_out/projection_1p5b_bal.json > gpurun_out/projection_bal.log 2>&1
grep -v '^ ' gpurun_out/projection_bal.log | grep schedule | tail -20
timeout 900 python tools/projection.py --model 1.5b --p 8 --out gpurun_out/projection_1p5b_even_p8.json > gpurun_out/projection_even.log 2>&1
grep -v '^ ' gpurun_out/projection_even.log | grep schedule | tail -6
