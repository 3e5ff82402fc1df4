timeout 900 python -m pytest tests -m gpu --timeout 300 -q 2>&1 | tail -2
timeout 700 python bench.py > gpurun_out/s_bench.log 2>&1
tail -1 gpurun_out/s_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['mfu'], d['clocks'])"
timeout 300 python -m tests.step_breakdown 2 32 > gpurun_out/s_breakdown.txt 2>&1; cat gpurun_out/s_breakdown.txt | head -8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'gemm_kernel|attn_' -c 6 -o gpurun_out/s_full -f python -m tests.prof_kernels > /dev/null 2>&1; ls gpurun_out/s_full.ncu-rep
