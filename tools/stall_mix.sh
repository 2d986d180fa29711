# ncu stall-reason mix (incl. no_instruction = instruction-cache misses) of one launch per regex
#   bash tools/stall_mix.sh name1 'regex1' skip1 [name2 'regex2' skip2 ...]
mkdir -p gpurun_out
while [ $# -ge 3 ]; do
  n=$1; r=$2; k=$3; shift 3
  timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:$r" -s $k -c 1 -o gpurun_out/sm_$n -f \
    python tools/profile_step.py --steps 3 > gpurun_out/sm_$n.log 2>&1
  ncu -i gpurun_out/sm_$n.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
d={}
for i,x in enumerate(h):
    if 'smsp__average_warps_issue_stalled' in x and 'per_issue_active' in x and 'not_issued' not in x:
        try: d[x.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')]=float(v[i])
        except: pass
dur=[v[i] for i,x in enumerate(h) if x=='gpu__time_duration.sum']
t=sum(d.values()) or 1
print('$n', dur, 'no_inst %.1f%%' % (100*d.get('no_instruction',0)/t), [(a, round(b,2)) for a,b in sorted(d.items(), key=lambda x:-x[1])[:5]])
" >> gpurun_out/stall_mix.txt
  rm -f gpurun_out/sm_$n.ncu-rep
done
