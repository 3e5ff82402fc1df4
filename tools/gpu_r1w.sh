# re-entry validation: full GPU suite, smoke, bench
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/w_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/w_pytest.log
tail -3 gpurun_out/w_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/w_bench.log 2>&1
tail -1 gpurun_out/w_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['clocks'])"
