timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x --timeout 300 -k "stream_k" 2>&1 | tail -3
timeout 300 python -m tests.bench_sk 2>&1 | tail -6
for v in 2 0; do PB_STREAMK=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ac_bench$v.log 2>&1
echo "PB_STREAMK=$v"; tail -1 gpurun_out/ac_bench$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"; done
