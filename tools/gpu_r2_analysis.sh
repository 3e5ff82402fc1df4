# Round-2 measured analysis on one B200: §8f rows on measured pass times and the 14B memory regime.
set -x
timeout 900 python -m pytest tests/test_executor_gpu.py -m gpu --timeout 600 -q -k "search_winner or solo or out_of_memory" > gpurun_out/r2e_pytest.log 2>&1; tail -3 gpurun_out/r2e_pytest.log
timeout 1500 python tools/measured_analysis.py --model 1.5b --p 8 --microbatches 32 --micro-batch 2 --schedules v-min v-half v-zb 1f1b zb-h1 --out gpurun_out/r2e_analysis_1p5b_p8.json --svg-prefix gpurun_out/r2e_gantt_1p5b_p8 > gpurun_out/r2e_analysis_1p5b.log 2>&1; tail -3 gpurun_out/r2e_analysis_1p5b.log
timeout 1500 python tools/measured_analysis.py --model 6b --p 8 --microbatches 32 --micro-batch 1 --schedules v-zb 1f1b v-half --out gpurun_out/r2e_analysis_6b_p8.json --svg-prefix gpurun_out/r2e_gantt_6b_p8 > gpurun_out/r2e_analysis_6b.log 2>&1; tail -3 gpurun_out/r2e_analysis_6b.log
timeout 2400 python tools/device_probe.py --model 14b --p 8 --microbatches 64 --micro-batch 4 --schedules v-min v-half --out gpurun_out/r2e_mem14b_mbs4_all.json > gpurun_out/r2e_mem14b_mbs4.log 2>&1; tail -2 gpurun_out/r2e_mem14b_mbs4.log
timeout 2400 python tools/device_probe.py --model 14b --p 8 --microbatches 128 --micro-batch 2 --schedules 1f1b --out gpurun_out/r2e_mem14b_1f1b_mbs2_m128.json > gpurun_out/r2e_mem14b_1f1b.log 2>&1; tail -2 gpurun_out/r2e_mem14b_1f1b.log
timeout 900 python tools/device_probe.py --model 14b --p 8 --microbatches 64 --micro-batch 5 --schedules v-min v-half v-zb 1f1b --devices 1,2 --out gpurun_out/r2e_mem14b_mbs5_dev12.json > gpurun_out/r2e_mem14b_mbs5.log 2>&1; grep '^{"schedule"' gpurun_out/r2e_mem14b_mbs5.log
ls gpurun_out | grep r2e_
