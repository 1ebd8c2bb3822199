#!/bin/bash
# NEXT-3 on hand-written kernels: parity, timing, launch list of one fit
python -m pytest tests/test_gpu_encode.py tests/test_gpu_parity.py -m gpu -x -q -k "encode or fit or adaptive or malformed" > gpurun_out/r2_fit_tests.log 2>&1; tail -3 gpurun_out/r2_fit_tests.log
python tools/profile_fit.py 2>&1 | tail -4
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_fit_launches.csv python tools/profile_fit.py > /dev/null 2>&1
python - <<'PY'
import csv,collections
rows=list(csv.reader(open("gpurun_out/r2_fit_launches.csv")))
hdr=None; agg=collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get("Metric Name")!="gpu__time_duration.sum": continue
        k=d["Kernel Name"][:90]; v=float(d["Metric Value"])
        a=agg.setdefault(k,[0,0.0]); a[0]+=1; a[1]+=v
for k,(n,t) in agg.items(): print(f"{n:4d} {t/1e3/n:10.1f} us/launch  {k}")
PY
