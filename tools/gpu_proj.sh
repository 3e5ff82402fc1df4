# p = 2/4/8 projections with the power-cap calibration -> gpurun_out/f4_proj_*
timeout 1500 python tools/projection.py --model 1.5b --p 2 4 8 --balance --out gpurun_out/f4_proj_1p5b_bal.json > gpurun_out/f4_proj_bal.log 2>&1
timeout 900 python tools/projection.py --model 1.5b --p 8 --out gpurun_out/f4_proj_1p5b_even_p8.json > gpurun_out/f4_proj_even.log 2>&1
timeout 1500 python tools/projection.py --model 6b --p 8 --microbatches 32 --micro-batch 1 --via-chunks --schedules 1f1b v-zb v-half zb-h1 --out gpurun_out/f4_proj_6b.json > gpurun_out/f4_proj6.log 2>&1
timeout 1500 python tools/projection.py --model 14b --p 8 --microbatches 64 --micro-batch 1 --via-chunks --schedules v-min 1f1b v-half --out gpurun_out/f4_proj_14b.json > gpurun_out/f4_proj14.log 2>&1
for f in gpurun_out/f4_proj_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['power_cap'])"; done
tail -3 gpurun_out/f4_proj14.log
