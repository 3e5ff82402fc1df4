PB_ATTN_FWD=3 timeout 300 python -m pytest tests/test_ops_gpu.py -q -x --timeout 120 -k "attention" 2>&1 | tail -2
for v in 3 1; do echo "PB_ATTN_FWD=$v"; PB_ATTN_FWD=$v timeout 300 python -m tests.bench_attn 2>&1 | grep batch | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['batch'],d['seq'],d['heads'],'fwd',round(d['fwd_tcgen05_tflops']),'bwd',round(d['bwd_tcgen05_tflops']))"; done
