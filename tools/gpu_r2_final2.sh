# Round-2 final GPU evidence (one B200) with the final kernels -> gpurun_out/r2g_*
set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2g_pytest.log 2>&1; tail -3 gpurun_out/r2g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; tail -1 gpurun_out/r2g_smoke.log
timeout 700 python bench.py > gpurun_out/r2g_bench.log 2>&1; tail -1 gpurun_out/r2g_bench.log | cut -c1-200
timeout 300 python -m tests.step_breakdown 2 32 > gpurun_out/r2g_breakdown.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 12000 -c 3200 --csv --log-file gpurun_out/r2g_launches.csv python bench.py --steps 1 --warmup 3 --microbatches 8 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'gemm_kernel|attn_|row_sumsq' -c 12 -o gpurun_out/r2g_full -f python -m tests.prof_kernels > /dev/null 2>&1
timeout 300 python -m tests.bench_attn > gpurun_out/r2g_attn.log 2>&1
timeout 600 python tools/host_overhead.py --model 1.5b --p 8 --microbatches 32 --micro-batch 2 --out gpurun_out/r2g_host_overhead.json > gpurun_out/r2g_host_overhead.log 2>&1; tail -2 gpurun_out/r2g_host_overhead.log
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py > gpurun_out/r2g_sanitize_$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/r2g_sanitize_$t.log; tail -2 gpurun_out/r2g_sanitize_$t.log
done
ls gpurun_out | grep r2g_
