cp tools/variants/lib_timers.so paper_2604_05885_b200/libjzknn.so
timeout 300 python tools/sweep.py 100000000 '[{"nmax0":128},{"nmax0":48}]'
