timeout 600 ncu --set full --clock-control none --import-source on -k regex:'gemm_kernel|attn_' -c 6 -o gpurun_out/r1_full -f python -m tests.prof_kernels > gpurun_out/i_ncu_full.log 2>&1
tail -2 gpurun_out/i_ncu_full.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 12000 -c 3200 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 3 --microbatches 8 --no-cpu-baseline > gpurun_out/i_ncu_launch.log 2>&1
tail -2 gpurun_out/i_ncu_launch.log
timeout 1500 python tools/projection.py --model 6b --p 8 --microbatches 32 --micro-batch 1 --via-chunks --schedules 1f1b v-zb v-half zb-h1 --out gpurun_out/projection_6b_p8.json > gpurun_out/proj6.log 2>&1
grep schedule gpurun_out/proj6.log | tail; tail -3 gpurun_out/proj6.log
timeout 1500 python tools/projection.py --model 14b --p 8 --microbatches 64 --micro-batch 1 --via-chunks --schedules v-min 1f1b v-half --out gpurun_out/projection_14b_p8.json > gpurun_out/proj14.log 2>&1
grep schedule gpurun_out/proj14.log | tail; tail -3 gpurun_out/proj14.log
