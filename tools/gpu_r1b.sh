set -x
python -m pytest tests/test_executor_gpu.py -x -q -k "isolate" 2>&1 | tail -5
python -m tests.bench_gemm 2048 > gpurun_out/bench_gemm_2048.txt 2>&1
python -m tests.bench_attn > gpurun_out/bench_attn.txt 2>&1
timeout 600 python bench.py --micro-batch 2 --microbatches 16 --no-cpu-baseline > gpurun_out/bench_mbs2.log 2>&1
timeout 900 python tools/projection.py --model 1.5b --p 2 4 8 --microbatches 32 --out gpurun_out/projection_1p5b.json > gpurun_out/projection.log 2>&1
tail -3 gpurun_out/bench_mbs2.log; grep -v '^ ' gpurun_out/projection.log | tail -20
