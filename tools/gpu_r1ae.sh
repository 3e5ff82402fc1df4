timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x --timeout 300 -k "pair_512 or forward_shape or backward_shape" 2>&1 | tail -3
timeout 300 python -m tests.bench_bm2 2>&1 | tail -8
for v in 1 0; do PB_GEMM_BM2=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ae_bench$v.log 2>&1
echo "PB_GEMM_BM2=$v"; tail -1 gpurun_out/ae_bench$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"; done
