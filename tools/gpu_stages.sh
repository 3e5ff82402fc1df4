timeout 300 python -m tests.bench_bm2 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['gemm'], d['r256_tflops'])"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/st6.log 2>&1
tail -1 gpurun_out/st6.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('6 stages', d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"
touch paper_2405_15362_b200/csrc/kernels/gemm_tc.cu; PB_NVCC_EXTRA=-DPB_GEMM_SMEM_KB=224 python -c "from paper_2405_15362_b200 import build as b; b.build()"
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x --timeout 300 2>&1 | tail -1
timeout 300 python -m tests.bench_bm2 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['gemm'], d['r256_tflops'])"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/st7.log 2>&1
tail -1 gpurun_out/st7.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('7 stages', d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"
