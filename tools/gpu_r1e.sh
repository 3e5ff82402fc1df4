B="timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline"
$B > gpurun_out/e_default.log 2>&1
PB_STREAMK=0 $B > gpurun_out/e_nosk.log 2>&1
PB_STREAMK=0 PB_ATTN_BWD=2 $B > gpurun_out/e_nosk_bwd2.log 2>&1
PB_STREAMK=0 PB_ATTN_BWD=2 PB_NO_FOLD=1 $B > gpurun_out/e_nosk_bwd2_nofold.log 2>&1
PB_STREAMK=0 timeout 300 python -m tests.step_breakdown 1 32 > gpurun_out/e_breakdown_nosk.txt 2>&1
for f in e_default e_nosk e_nosk_bwd2 e_nosk_bwd2_nofold; do echo $f; tail -1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"; done
cat gpurun_out/e_breakdown_nosk.txt
