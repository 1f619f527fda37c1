bash tools/variants/run2.sh vec vec2 ipt8 ipt12 2>&1 | grep -v JZ_STATS
cp tools/variants/lib_vec2.so paper_2604_05885_b200/libjzknn.so
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
