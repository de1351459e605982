# usage: bash scripts/gpu_profile.sh TAG [CONFIG]
# Launch list (cold-cache, serialised) of a short bench run + one `ncu --set full` capture of the deposit kernel.
TAG=${1:-r01}; CFG=${2:-C4}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"deposit|pixel_window|tile_kernel|fit_kernel" \
   --log-file gpurun_out/${TAG}_launches.csv python bench.py --config $CFG --steps 2 --warmup 1 --e2e-steps 1 \
   --no-cpu-baseline > gpurun_out/${TAG}_launches_bench.json 2> gpurun_out/${TAG}_launches_bench.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:deposit -s 1 -c 1 \
   -o gpurun_out/${TAG}_deposit python bench.py --config $CFG --steps 1 --warmup 1 --e2e-steps 0 \
   --no-cpu-baseline > gpurun_out/${TAG}_full_bench.json 2> gpurun_out/${TAG}_full_bench.err
ls -la gpurun_out/
