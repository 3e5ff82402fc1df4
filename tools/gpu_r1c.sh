set -x
T="--timeout 420"
python -m pytest tests/test_gemm_gpu.py tests/test_ops_gpu.py $T -x -q 2>&1 | tail -8
python -m pytest tests/test_executor_gpu.py tests/test_multiprocess_gpu.py $T -x -q 2>&1 | tail -8
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python -m tests.bench_gemm 2048 > gpurun_out/bench_gemm_2048_sk.txt 2>&1
python -m tests.bench_attn > gpurun_out/bench_attn_c.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_c.log 2>&1
timeout 300 python -m tests.step_breakdown 1 32 > gpurun_out/breakdown_c.txt 2>&1
tail -1 gpurun_out/bench_c.log | cut -c1-400; cat gpurun_out/breakdown_c.txt
timeout 1000 python tools/projection.py --model 1.5b --p 2 4 8 --microbatches 32 --out gpurun_out/projection_1p5b.json > gpurun_out/projection.log 2>&1
grep -v '^ ' gpurun_out/projection.log | tail -20
