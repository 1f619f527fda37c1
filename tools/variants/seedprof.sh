# diag-walk counters at 10^7 / 10^8, then source-attributed ncu of the seeded (ideal-threshold) k_leaf at 10^7
cp paper_2604_05885_b200/libjzknn.so /tmp/lib_orig.so
cp tools/variants/lib_diagw.so paper_2604_05885_b200/libjzknn.so
for n in 10000000 100000000; do timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --n $n 2>&1 | grep JZ_DIAG | tail -1; done
cp tools/variants/lib_seed.so paper_2604_05885_b200/libjzknn.so
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_leaf -s 2 -c 1 -o gpurun_out/l2l_seed python tools/seed_exp.py 10000000 > gpurun_out/prof_seed.log 2>&1
ncu -i gpurun_out/l2l_seed.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/l2l_seed_cs.csv 2>&1
python tools/src_cats.py gpurun_out/l2l_seed_cs.csv
python tools/ncu_summary.py gpurun_out/l2l_seed.ncu-rep | head -30
cp /tmp/lib_orig.so paper_2604_05885_b200/libjzknn.so
