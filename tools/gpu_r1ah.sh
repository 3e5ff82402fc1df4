timeout 600 python -m pytest tests/test_ops_gpu.py tests/test_executor_gpu.py -q -x --timeout 300 2>&1 | tail -2
timeout 300 python -m tests.bench_attn 2>&1 | grep batch | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['batch'],d['seq'],d['heads'],'fwd',round(d['fwd_tcgen05_tflops']),'bwd',round(d['bwd_tcgen05_tflops']))"
for v in 0 1; do PB_ATTN_FWD=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ah_bench$v.log 2>&1
echo "PB_ATTN_FWD=$v"; tail -1 gpurun_out/ah_bench$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"; done
