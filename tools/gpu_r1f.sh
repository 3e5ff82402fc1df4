timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_ops_gpu.py --timeout 120 -q 2>&1 | tail -4
timeout 300 python -m tests.bench_attn > gpurun_out/f_bench_attn.txt 2>&1
B="timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline"
$B > gpurun_out/f_default.log 2>&1
PB_ATTN_BWD=2 $B > gpurun_out/f_bwd2.log 2>&1
for f in f_default f_bwd2; do echo $f; tail -1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"; done
head -4 gpurun_out/f_bench_attn.txt
timeout 300 ncu --set full --clock-control none -k regex:'gemm_kernel|nvjet|xmma|cutlass|sm100' -s 4 -c 2 -o gpurun_out/gemm_cmp -f python -m tests.prof_gemm_cmp > gpurun_out/f_ncu_cmp.log 2>&1
tail -3 gpurun_out/f_ncu_cmp.log
