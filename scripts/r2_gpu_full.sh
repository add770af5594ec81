# full GPU suite + smoke
timeout 2400 python -m pytest tests/ -q -m gpu --timeout 900 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
