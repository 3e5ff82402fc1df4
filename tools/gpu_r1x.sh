# knobs re-check: micro-batch 4, stream-K in-step, per-shape GEMM TFLOP/s
timeout 300 python -m tests.bench_gemm 4096 > gpurun_out/x_gemm.log 2>&1; cat gpurun_out/x_gemm.log | cut -c1-200
for cfg in "--micro-batch 4 --microbatches 16" "--micro-batch 2 --microbatches 32"; do
timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline $cfg > gpurun_out/x_bench.log 2>&1
echo "$cfg"; tail -1 gpurun_out/x_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"
done
PB_STREAMK=1 timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/x_bench_sk.log 2>&1
echo streamk; tail -1 gpurun_out/x_bench_sk.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"
