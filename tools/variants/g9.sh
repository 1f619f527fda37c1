mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  for c in knn xq fof dist; do
    timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_case.py $c > gpurun_out/san/${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(tail -2 gpurun_out/san/${tool}_${c}.log | tr '\n' ' ')"
  done
done
