T=${TAG:-r02zf}
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "fused_profile or depth_profile or both or row_path or c1_full" > gpurun_out/${T}_pytest.log 2>&1; tail -3 gpurun_out/${T}_pytest.log; grep -E "^E " gpurun_out/${T}_pytest.log | head -5
timeout 600 python scripts/profile_fusion.py C4 C5 > gpurun_out/${T}_profile_fusion.jsonl 2> gpurun_out/${T}_profile_fusion.err; cat gpurun_out/${T}_profile_fusion.jsonl; tail -3 gpurun_out/${T}_profile_fusion.err
timeout 120 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/${T}_bench.json')); print('C4', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))"
