# attention bwd v4: parity, throughput vs v3, trace
timeout 300 python -m pytest tests/test_ops_gpu.py -q -x --timeout 120 -k "attn or attention" 2>&1 | tail -3
for v in 4 3; do echo "PB_ATTN_BWD=$v"; PB_ATTN_BWD=$v timeout 300 python -m tests.bench_attn 2>&1 | grep batch | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['batch'],d['seq'],d['heads'],'fwd',round(d['fwd_tcgen05_tflops']),'bwd',round(d['bwd_tcgen05_tflops']))"; done
touch paper_2405_15362_b200/csrc/kernels/attention_tc.cu
PB_ATTN_TRACE_BUILD=1 python -c "from paper_2405_15362_b200 import build as b; b.build()" 2>&1 | tail -2
PB_ATTN_TRACE=1 timeout 120 python -m tests.trace_attn_bwd > gpurun_out/z_trace.log 2>&1; tail -16 gpurun_out/z_trace.log
