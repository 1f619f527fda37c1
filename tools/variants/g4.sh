timeout 900 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -15
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sort_fixup" 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python tools/dist_phases.py 100000000 8 2>&1 | tail -80
