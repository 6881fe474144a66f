ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01ai_err.csv python tools/fault_times.py > gpurun_out/r01ai.log 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open("gpurun_out/r01ai_err.csv")) if len(r)>10]
hdr=rows[0]; ki=hdr.index("Kernel Name"); vi=hdr.index("Metric Value"); ui=hdr.index("Metric Unit")
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows[1:]:
    name=r[ki].split("(")[0][-50:]
    v=float(r[vi].replace(",",""))*(1e-3 if r[ui] in ("nsecond","ns") else 1)
    agg[name][0]+=1; agg[name][1]+=v
for k,(n,t) in sorted(agg.items(), key=lambda x:-x[1][1])[:25]:
    print(f"{t:10.1f} us  {n:4d}x  {k}")
PY
