timeout 300 python -m pytest tests/test_ops_gpu.py --timeout 120 -q 2>&1 | tail -3
timeout 300 python -m tests.bench_attn 2>&1 | grep batch
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/k_bench.log 2>&1
tail -1 gpurun_out/k_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"
timeout 300 ncu --set full --clock-control none -k regex:'attn_' -c 3 -o gpurun_out/attn_k -f python -m tests.prof_kernels > /dev/null 2>&1; ls gpurun_out/attn_k.ncu-rep
