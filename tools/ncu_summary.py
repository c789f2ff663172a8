"""Summarise an ncu report (--page raw) into the JSON fields profiles/ quotes."""
import csv, sys, subprocess, io, json
rep=sys.argv[1]
txt=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
rows=list(csv.reader(io.StringIO(txt)))
hdr=rows[0]; units=rows[1]; idx={h:i for i,h in enumerate(hdr)}
want=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','sm__throughput.avg.pct_of_peak_sustained_elapsed','sm__cycles_active.avg','gpc__cycles_elapsed.max','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__grid_size','launch__block_size','smsp__issue_active.avg.pct_of_peak_sustained_active','l1tex__throughput.avg.pct_of_peak_sustained_active','lts__throughput.avg.pct_of_peak_sustained_elapsed','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','smsp__cycles_active.avg']
out=[]
for r in rows[2:]:
    d={}
    for w in want:
        if w in idx: d[w]=r[idx[w]]+(' '+units[idx[w]] if units[idx[w]] else '')
    out.append(d)
print(json.dumps(out,indent=1))
