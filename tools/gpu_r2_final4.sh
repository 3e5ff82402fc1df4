# Round-2 closing evidence after the forward-softmax and norm-backward changes -> gpurun_out/r2y_*
set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2y_pytest.log 2>&1; tail -3 gpurun_out/r2y_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2y_smoke.log 2>&1; tail -1 gpurun_out/r2y_smoke.log
timeout 700 python bench.py > gpurun_out/r2y_bench.log 2>&1; tail -1 gpurun_out/r2y_bench.log | cut -c1-200
timeout 300 python -m tests.step_breakdown 2 32 > gpurun_out/r2y_breakdown.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 12000 -c 3200 --csv --log-file gpurun_out/r2y_launches.csv python bench.py --steps 1 --warmup 3 --microbatches 8 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'gemm_kernel|attn_|row_sumsq' -c 12 -o gpurun_out/r2y_full -f python -m tests.prof_kernels > /dev/null 2>&1
timeout 300 python -m tests.bench_attn > gpurun_out/r2y_attn.log 2>&1
timeout 300 python -m tests.bench_gemm 4096 > gpurun_out/r2y_gemm.log 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py > gpurun_out/r2y_sanitize_$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/r2y_sanitize_$t.log; tail -2 gpurun_out/r2y_sanitize_$t.log
done
ls gpurun_out | grep r2y_
