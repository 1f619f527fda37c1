cp tools/variants/lib_seed.so paper_2604_05885_b200/libjzknn.so
for n in 10000000 100000000; do for nm in 0 64 48; do timeout 300 python tools/seed_exp.py $n $nm 2>&1 | tail -1; done; done
