B="timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline"
$B --micro-batch 2 --microbatches 16 > gpurun_out/g_mbs2.log 2>&1
$B --micro-batch 4 --microbatches 8 > gpurun_out/g_mbs4.log 2>&1
for f in g_mbs2 g_mbs4; do echo $f; tail -1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"; done
timeout 1500 python tools/projection.py --model 1.5b --p 2 4 8 --microbatches 32 --out gpurun_out/projection_1p5b.json > gpurun_out/projection.log 2>&1
grep -v '^ ' gpurun_out/projection.log | tail -20
