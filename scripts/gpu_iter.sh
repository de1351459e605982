# one GPU iteration: smoke, GPU tests, short bench, profile (TAG)
TAG=${1:-iter}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-budget-s 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -3 gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:deposit_fast -s 1 -c 1 \
   -o gpurun_out/${TAG}_deposit python bench.py --config C4 --steps 1 --warmup 1 --e2e-steps 0 \
   --no-cpu-baseline > /dev/null 2> gpurun_out/${TAG}_ncu.err; tail -2 gpurun_out/${TAG}_ncu.err
