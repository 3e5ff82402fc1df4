timeout 300 python -m pytest tests/test_ops_gpu.py --timeout 120 -q -x 2>&1 | tail -1
for i in 1 2; do timeout 300 python -m tests.bench_attn 2>&1 | grep batch | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['batch'],d['seq'],d['heads'],'fwd',round(d['fwd_tcgen05_tflops']),'bwd',round(d['bwd_tcgen05_tflops']))"; done
