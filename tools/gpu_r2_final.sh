# Round-2 GPU evidence (one B200) -> gpurun_out/r2f_*: sanitizers, step breakdown, ncu launch list + full
# capture, attention vs SDPA, §8f measured analysis (1.5B / 6B at p=8), bench.
set -x
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py > gpurun_out/r2f_sanitize_$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/r2f_sanitize_$t.log; tail -4 gpurun_out/r2f_sanitize_$t.log
done
timeout 300 python -m tests.step_breakdown 2 32 > gpurun_out/r2f_breakdown.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 12000 -c 3200 --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 1 --warmup 3 --microbatches 8 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'gemm_kernel|attn_|row_sumsq' -c 12 -o gpurun_out/r2f_full -f python -m tests.prof_kernels > /dev/null 2>&1
timeout 300 python -m tests.bench_attn > gpurun_out/r2f_attn.log 2>&1
timeout 1500 python tools/measured_analysis.py --model 1.5b --p 8 --microbatches 32 --micro-batch 2 --schedules v-min v-half v-zb 1f1b zb-h1 --out gpurun_out/r2f_analysis_1p5b_p8.json --svg-prefix gpurun_out/r2f_gantt_1p5b_p8 > gpurun_out/r2f_analysis_1p5b.log 2>&1; tail -3 gpurun_out/r2f_analysis_1p5b.log
timeout 1500 python tools/measured_analysis.py --model 6b --p 8 --microbatches 32 --micro-batch 1 --schedules v-zb 1f1b v-half --out gpurun_out/r2f_analysis_6b_p8.json --svg-prefix gpurun_out/r2f_gantt_6b_p8 > gpurun_out/r2f_analysis_6b.log 2>&1; tail -3 gpurun_out/r2f_analysis_6b.log
timeout 700 python bench.py > gpurun_out/r2f_bench.log 2>&1
ls gpurun_out | grep r2f_
