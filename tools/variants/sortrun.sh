for v in "$@"; do
  cp tools/variants/lib_$v.so paper_2604_05885_b200/libjzknn.so
  timeout 300 python tools/sweep.py 100000000 '[{"nmax0":128}]' 2>&1 | sed "s/^/$v /" | tail -1
done
