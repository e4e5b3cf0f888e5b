# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -v "^\.\+ *\[" | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
