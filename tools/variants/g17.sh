for mode in ghost all; do
if [ $mode = all ]; then export JZ_REWALK_ALL=1; fi
JZ_TIMING=1 JZ_REPS=2 JZ_PROF_LAST=1 timeout 900 python tools/dist_phases.py 100000000 8 > /tmp/o.json 2> /tmp/e.txt
echo "== $mode"; sed -n '/---- last rep/,$p' /tmp/e.txt | grep "^rank [0]" | grep -v "exchange\|gather boxes\|allreduce"
python -c "
import json; d=json.load(open('/tmp/o.json')); print({k:v for k,v in d.items() if k!='ranks'}); [print(r['rank'], r['local'], round(r['ghost_frac'],3), round(r['requery_frac'],3), round(r['busy_ms'],1)) for r in d['ranks']]"
cp /tmp/o.json gpurun_out/dist_phases_$mode.json
done
