# Round-end GPU refresh (one B200): GPU tests, smoke, bench, step breakdown, ncu launch list + full capture, attention table, projections (1.5B/6B/14B, and the LM-head-balanced 30/31-layer variants) -> gpurun_out/f7_*
set -x
timeout 1200 python -m pytest tests -m gpu --timeout 300 -q > gpurun_out/f7_pytest.log 2>&1; tail -3 gpurun_out/f7_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 700 python bench.py > gpurun_out/f7_bench.log 2>&1
tail -1 gpurun_out/f7_bench.log | cut -c1-300
timeout 300 python -m tests.step_breakdown 2 32 > gpurun_out/f7_breakdown.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 12000 -c 3200 --csv --log-file gpurun_out/f7_launches.csv python bench.py --steps 1 --warmup 3 --microbatches 8 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'gemm_kernel|attn_' -c 7 -o gpurun_out/f7_full -f python -m tests.prof_kernels > /dev/null 2>&1
timeout 300 python -m tests.bench_attn > gpurun_out/f7_attn.log 2>&1
timeout 1500 python tools/projection.py --model 1.5b --p 2 4 8 --balance --out gpurun_out/f7_proj_1p5b_bal.json > gpurun_out/f7_proj_bal.log 2>&1
timeout 900 python tools/projection.py --model 1.5b --p 8 --out gpurun_out/f7_proj_1p5b_even_p8.json > gpurun_out/f7_proj_even.log 2>&1
timeout 1500 python tools/projection.py --model 6b --p 8 --microbatches 32 --micro-batch 1 --via-chunks --schedules 1f1b v-zb v-half zb-h1 --out gpurun_out/f7_proj_6b.json > gpurun_out/f7_proj6.log 2>&1
timeout 1500 python tools/projection.py --model 14b --p 8 --microbatches 64 --micro-batch 1 --via-chunks --schedules v-min 1f1b v-half --out gpurun_out/f7_proj_14b.json > gpurun_out/f7_proj14.log 2>&1
ls -la gpurun_out | tail -25
timeout 1500 python tools/projection.py --model 6b --layers 31 --p 8 --microbatches 32 --micro-batch 1 --via-chunks --schedules 1f1b v-zb v-half zb-h1 --out gpurun_out/f7_proj_6b_l31.json > gpurun_out/f7_proj6_l31.log 2>&1
timeout 1500 python tools/projection.py --model 14b --layers 31 --p 8 --microbatches 64 --micro-batch 1 --via-chunks --schedules 1f1b v-zb v-half v-min --out gpurun_out/f7_proj_14b_l31.json > gpurun_out/f7_proj14_l31.log 2>&1
timeout 1500 python tools/projection.py --model 1.5b --layers 30 --p 8 --balance --out gpurun_out/f7_proj_1p5b_l30_bal.json > gpurun_out/f7_proj_l30.log 2>&1
ls gpurun_out | grep f7_
