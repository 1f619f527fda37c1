cp paper_2604_05885_b200/libjzknn.so /tmp/lib_orig.so
for v in nopersist persist; do cp tools/variants/lib_$v.so paper_2604_05885_b200/libjzknn.so; echo $v; E2E_REPS=6 python tools/e2e_probe.py 2>&1 | grep knn_host; done
cp /tmp/lib_orig.so paper_2604_05885_b200/libjzknn.so
