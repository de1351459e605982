python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "general_wire or forced_table" 2>&1 | grep -E "passed|failed|Error|assert" | head -8
