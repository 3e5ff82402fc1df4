timeout 300 python -m pytest tests/test_ops_gpu.py --timeout 120 -q -x 2>&1 | tail -2
PB_ATTN_TRACE_FWD=1 timeout 120 python -m tests.trace_attn_fwd 2>&1 | tail -3
PB_ATTN_TRACE=1 timeout 120 python -m tests.trace_attn_bwd 2>&1 | tail -3
timeout 300 python -m tests.bench_attn 2>&1 | grep batch | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['batch'],d['seq'],d['heads'],'fwd',round(d['fwd_tcgen05_tflops']),'bwd',round(d['bwd_tcgen05_tflops']))"
