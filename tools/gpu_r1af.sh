timeout 1500 python -m pytest tests -m gpu --timeout 300 -q > gpurun_out/af_pytest.log 2>&1; tail -3 gpurun_out/af_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 700 python bench.py > gpurun_out/af_bench.log 2>&1
tail -1 gpurun_out/af_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['clocks'], d['cpu_baseline']['value'])"
