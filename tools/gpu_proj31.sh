# 31-layer variants: 2 layers per V stage, 1 on the LM-head stage (the head ~ one layer): balanced devices
timeout 1500 python tools/projection.py --model 6b --layers 31 --p 8 --microbatches 32 --micro-batch 1 --via-chunks --schedules 1f1b v-zb v-half zb-h1 --out gpurun_out/f5_proj_6b_l31.json > gpurun_out/f5_proj6.log 2>&1
timeout 1500 python tools/projection.py --model 14b --layers 31 --p 8 --microbatches 64 --micro-batch 1 --via-chunks --schedules 1f1b v-zb v-half v-min --out gpurun_out/f5_proj_14b_l31.json > gpurun_out/f5_proj14.log 2>&1
for f in gpurun_out/f5_proj_*.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['power_cap']['factor'],3)); [print(r['schedule'], r['p'], round(r['projected_tokens_per_s']/1e3,1), round(r.get('tokens_per_s_vs_1f1b',0),3), round(r['bubble_rate'],3), round(r['pipeline_roofline_frac'],3), round(r['max_pool_gib'],2), round(r.get('pool_vs_1f1b',0),2), r['target_stage_layers']) for r in d['runs']]"; done
tail -3 gpurun_out/f5_proj14.log
