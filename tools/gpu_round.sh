#!/bin/bash
# one gpurun session: tests, bench, launch list, source-attributed ncu of k_leaf; $1 = tag
tag=${1:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gputests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/${tag}_gputests.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
cat gpurun_out/${tag}_bench.json | head -c 3000
if [ "$2" = "src" ]; then
  bash tools/prof_src.sh ${tag}
  python tools/src_lines.py gpurun_out/l2l_${tag}_cs.csv 60 > gpurun_out/l2l_${tag}_lines.txt 2>&1
  head -70 gpurun_out/l2l_${tag}_lines.txt
fi
