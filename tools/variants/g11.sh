timeout 900 python -m pytest tests -m gpu -x -q -k "fof" 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for v in fofold fofnew fofnofull; do cp tools/variants/lib_$v.so paper_2604_05885_b200/libjzknn.so; echo "== $v"; timeout 600 python tools/fof_bench.py 100000000 2>&1 | tail -3; done
cp tools/variants/lib_fofnew.so paper_2604_05885_b200/libjzknn.so
