"""Instruction and stall shares of k_sig (k_distribute.cu) by pass-1 phase, from an ncu report's
source page.  usage: python tools/ncu_phases.py REPORT.ncu-rep"""
import csv, io, subprocess, sys, collections
rep=sys.argv[1]
out=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","cuda,sass"],capture_output=True,text=True).stdout
hdr=None; fpath=None; cur=None; agg=collections.Counter(); st=collections.Counter()
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0]=="File Path": fpath=row[1]; continue
    if row[0]=="Function Name": continue
    if row[0]=="Line No": hdr=row; continue
    if hdr is None: continue
    d=dict(zip(hdr,row)); addr=d.get("Address","")
    if row[0].strip().isdigit() and not addr:
        cur=(fpath,int(row[0])); continue
    if row[0].strip().isdigit(): cur=(fpath,int(row[0]))
    try:
        agg[cur]+=int(float(d.get("Instructions Executed","0") or 0)); st[cur]+=int(float(d.get("Warp Stall Sampling (All Samples)","0") or 0))
    except ValueError: pass
bounds=[(154,"A encode"),(230,"B read starts"),(241,"validity"),(254,"C p-mer keys"),(312,"D/E sliding min"),(386,"F runs"),(422,"G emission"),(532,"carry"),(547,"stats"),(10**9,"end")]
ph=collections.Counter(); phs=collections.Counter()
T=sum(agg.values()); S=sum(st.values())
for (f,l),v in agg.items():
    if f and f.endswith("k_distribute.cu"):
        name="pre"
        for (b,n),(b2,_) in zip(bounds,bounds[1:]):
            if b<=l<b2: name=n
    else: name="helpers:"+(f or "?").split("/")[-1]
    ph[name]+=v; phs[name]+=st[(f,l)]
for n,v in sorted(ph.items(), key=lambda x:-x[1]): print(f"{n:28s} instr {100*v/T:5.1f}%  stalls {100*phs[n]/S:5.1f}%")
