# attention bwd phase trace at the bench shape
touch paper_2405_15362_b200/csrc/kernels/attention_tc.cu
PB_ATTN_TRACE_BUILD=1 python -c "from paper_2405_15362_b200 import build as b; b.build()" 2>&1 | tail -2
PB_ATTN_TRACE=1 timeout 120 python -m tests.trace_attn_bwd > gpurun_out/y_trace.log 2>&1; tail -40 gpurun_out/y_trace.log
