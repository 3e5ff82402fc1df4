timeout 120 python -m tests.prof_sk
timeout 300 ncu --set full --clock-control none -k regex:gemm_kernel -s 2 -c 2 -o gpurun_out/sk_cmp -f python -m tests.prof_sk > gpurun_out/j_ncu.log 2>&1
tail -2 gpurun_out/j_ncu.log
