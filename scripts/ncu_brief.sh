# brief of one .ncu-rep: duration, issue, stalls, opcode mix (per element when N given)
rep=$1; n=${2:-}
ncu -i $rep --page raw --csv 2>/dev/null > /tmp/_raw.csv
python3 - <<'PY'
import csv
rows=list(csv.reader(open('/tmp/_raw.csv')))
h=rows[0]; v=rows[2]
for k,x in zip(h,v):
    if ('smsp__average_warps_issue_stalled' in k and 'ratio' in k) or k in ('gpu__time_duration.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','launch__grid_size','dram__bytes_read.sum','dram__bytes_write.sum'):
        try:
            if float(x)>0.05: print(f"  {k} {x}")
        except: pass
PY
ncu -i $rep --page source --csv --print-source sass 2>/dev/null > /tmp/_sass.csv
if [ -n "$n" ]; then python3 $(dirname $0)/sass_mix.py /tmp/_sass.csv --elems $n | head -25; else python3 $(dirname $0)/sass_mix.py /tmp/_sass.csv | head -25; fi
