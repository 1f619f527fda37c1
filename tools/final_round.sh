# round-end evidence in one GPU session: GPU tests, default bench, launch list + k_leaf ncu + build
# DRAM (tools/prof_r02.sh), smoke, FoF at 10^8, compute-sanitizer on small cases. $1 = tag
tag=${1:-r02z}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gputests.log 2>&1; echo "tests: $(tail -1 gpurun_out/${tag}_gputests.log)"
timeout 900 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err; echo "bench rc=$?"
bash tools/prof_r02.sh ${tag} > /dev/null 2>&1; echo "prof done"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo "smoke: $(tail -1 gpurun_out/smoke_${tag}.log)"
timeout 600 python tools/fof_bench.py 100000000 > gpurun_out/fof_${tag}.json 2> /dev/null; echo "fof rc=$?"
bash tools/sanitize.sh > gpurun_out/sanitize_${tag}.txt 2>&1; cat gpurun_out/sanitize_${tag}.txt
