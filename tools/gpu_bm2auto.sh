timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x --timeout 300 2>&1 | tail -1
for v in auto 0 auto 0; do
if [ $v = auto ]; then unset PB_GEMM_BM2; else export PB_GEMM_BM2=0; fi
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bm_$v.log 2>&1
echo "BM2=$v"; tail -1 gpurun_out/bm_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'], d['loss'])"
done
