# one ncu --set full capture of the deposit kernel for a config (default build or DAXM_LIBRARY)
TAG=${1:-n}; CFG=${2:-C4}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:deposit -s 1 -c 1 \
   -o gpurun_out/${TAG} python bench.py --config $CFG --steps 1 --warmup 1 --e2e-steps 0 \
   --no-cpu-baseline > /dev/null 2> gpurun_out/${TAG}.err; tail -2 gpurun_out/${TAG}.err
