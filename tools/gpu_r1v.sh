timeout 300 python -m pytest tests/test_ops_gpu.py tests/test_gemm_gpu.py --timeout 120 -q -x 2>&1 | tail -1
timeout 300 python -m tests.bench_attn 2>&1 | grep batch | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['batch'],d['seq'],d['heads'],'fwd',round(d['fwd_tcgen05_tflops']),'bwd',round(d['bwd_tcgen05_tflops']))"
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/v_bench.log 2>&1
tail -1 gpurun_out/v_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"
