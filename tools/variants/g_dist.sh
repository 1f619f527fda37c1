P="import json,sys; d=json.load(sys.stdin); print({k:v for k,v in d.items() if k!='ranks'}); [print(r['rank'], round(r['busy_ms'],1), {k:round(v,1) for k,v in r['phase_wall_ms'].items()}) for r in d['ranks']]"
cp paper_2604_05885_b200/libjzknn.so /tmp/lib_orig.so
for v in s5 orig; do
  [ $v = s5 ] && cp tools/variants/lib_s5.so paper_2604_05885_b200/libjzknn.so
  [ $v = orig ] && cp /tmp/lib_orig.so paper_2604_05885_b200/libjzknn.so
  for rep in 1 2; do echo "$v rep $rep"; JZ_SKIP_T1=1 timeout 600 python tools/dist_phases.py 100000000 8 2>/dev/null | python -c "$P"; done
done
