# variants bench + lock tests + full GPU suite
bash scripts/gpu_variants.sh
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "lock or c1_full or c2_full or single_bin" 2>&1 | tail -4
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
