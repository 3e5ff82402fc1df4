set -x
timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_ops_gpu.py --timeout 120 -q 2>&1 | tail -8
timeout 900 python -m pytest tests/test_executor_gpu.py tests/test_multiprocess_gpu.py --timeout 240 -q 2>&1 | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 python -m tests.bench_gemm 2048 > gpurun_out/bench_gemm_2048_sk.txt 2>&1
timeout 300 python -m tests.bench_attn > gpurun_out/bench_attn_d.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_d.log 2>&1
timeout 300 python -m tests.step_breakdown 1 32 > gpurun_out/breakdown_d.txt 2>&1
tail -1 gpurun_out/bench_d.log | cut -c1-600; cat gpurun_out/breakdown_d.txt; cat gpurun_out/bench_attn_d.txt; cat gpurun_out/bench_gemm_2048_sk.txt
