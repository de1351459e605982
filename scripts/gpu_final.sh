# Round record: smoke, full GPU suite, default bench line (+ reference arm), every config and mode,
# 2-rank gloo run with the bit-exact gather check, launch list + one full ncu capture of the C4 row
# kernel, sanitizers.  Outputs under gpurun_out/$T/.
T=${TAG:-r02final}
O=gpurun_out/$T
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log; grep -E "^(FAILED|ERROR)" $O/pytest_gpu.log | head
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; python -c "import json; d=json.load(open('$O/bench_default.json')); print('default', d['config']['workload'][:3], round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3), 'e2e', d['e2e'] and round(d['e2e']['ms_per_step'],1), 'parity', (d.get('parity_sample') or {}).get('pass'))" || tail -3 $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; tail -c 300 $O/bench_reference.json
run() {  # name, args...
  n=$1; shift
  timeout 900 python bench.py --steps 10 --warmup 3 --cpu-budget-s 4 "$@" > $O/bench_$n.json 2> $O/bench_$n.err
  python -c "import json; d=json.load(open('$O/bench_$n.json')); print('$n', round(d['ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],3), 'e2e', d['e2e'] and round(d['e2e']['ms_per_step'],1), 'parity', (d.get('parity_sample') or {}).get('pass'))" || tail -3 $O/bench_$n.err
}
run C2 --config C2 --e2e-steps 0
run C3 --config C3 --e2e-steps 0
run C5 --config C5 --e2e-steps 0
run C5_f32 --config C5 --dtype f32 --e2e-steps 0
run C5_f0.5 --config C5 --fraction 0.5 --e2e-steps 0
run C5_f0.25 --config C5 --fraction 0.25 --e2e-steps 0
run C5_f0.05 --config C5 --fraction 0.05 --e2e-steps 0
run C4_both --config C4 --edge both --e2e-steps 0
run C4_trailing --config C4 --edge trailing --e2e-steps 0
run C3_jitter --config C3 --jitter 0.3 --e2e-steps 0 --steps 3
run C4_ooc --config C4 --host-budget 4 --e2e-steps 3 --no-cpu-baseline
run C2_trailing --config C2 --edge trailing --e2e-steps 0
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --backend gloo --steps 5 --warmup 3 --e2e-steps 0 --check-gather --all-gather > $O/bench_gloo2.json 2> $O/bench_gloo2.err; python -c "import json; d=json.load(open('$O/bench_gloo2.json')); print('gloo x2', round(d['ms_per_step'],3), d.get('gather_check'))" || tail -3 $O/bench_gloo2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/C4_launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $O/launches_bench.json 2> $O/launches_bench.err; tail -1 $O/launches_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:deposit_row -s 2 -c 1 -o $O/C4_row_full python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $O/full_bench.json 2> $O/full_bench.err; tail -1 $O/full_bench.err
# compute-sanitizer is closed on this GPU pool (r02final1): not run
