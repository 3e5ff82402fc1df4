timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_ops_gpu.py --timeout 120 -q -x 2>&1 | tail -2
timeout 300 ncu --set full --clock-control none -k regex:'gemm_kernel' -c 3 -o gpurun_out/o_gemm -f python -m tests.prof_kernels > /dev/null 2>&1
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/o_bench.log 2>&1
tail -1 gpurun_out/o_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"
