T=${TAG:-r02s2t}
timeout 300 python scripts/row_stats.py C1 C2 C3 C4 C5 C4:trailing 2>&1 | tail -6 | python -c "
import sys, json
for l in sys.stdin:
    n, _, j = l.partition(' ')
    try: d = json.loads(j); print(n, 'prepass_ms', round(d['prepass_ms'],1), 'row_path', d['row_path'], 'small', d['small'], 'general', d['general'])
    except Exception: print(l[:200])"
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; tail -2 gpurun_out/${T}_pytest_gpu.log; grep -E "^E |FAILED" gpurun_out/${T}_pytest_gpu.log | head -5
timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_C4.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/${T}_C4.json')); print('C4', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), 'prepass', round(d['prepass_ms'],1))"
