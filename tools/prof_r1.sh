set -x
python -m tests.step_breakdown 1 32 > gpurun_out/breakdown_m32.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 15500 -c 5200 --csv --log-file gpurun_out/launches_m8.csv python bench.py --steps 1 --warmup 3 --microbatches 8 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 3 -o gpurun_out/gemm_full -f python -m tests.prof_kernels > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_ -c 3 -o gpurun_out/attn_full -f python -m tests.prof_kernels > gpurun_out/ncu_attn.log 2>&1
ls -la gpurun_out
