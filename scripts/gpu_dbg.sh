python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python scripts/debug_m1.py 2>&1 | tail -8
