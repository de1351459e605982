# final verification of the committed state: smoke, full GPU suite, default bench line, reference arm
T=${TAG:-r02verify}
O=gpurun_out/$T
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log; grep -E "^(FAILED|ERROR)" $O/pytest_gpu.log | head
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; python -c "import json; d=json.load(open('$O/bench_default.json')); print('default', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3), 'traffic', d['roofline']['traffic'], 'e2e', round(d['e2e']['ms_per_step'],1), 'parity', (d.get('parity_sample') or {}).get('pass'), 'launches', d.get('gpu_launches'))" || tail -3 $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; tail -c 200 $O/bench_reference.json
