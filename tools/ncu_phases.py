"""Instruction and stall shares of k_sig (k_distribute.cu) by pass-1 phase, from an ncu report's
source page.  usage: python tools/ncu_phases.py REPORT.ncu-rep"""
import csv, io, os, subprocess, sys, collections
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
# phase boundaries from the markers in the current source (line numbers move with edits)
SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1407_1507_b200", "csrc", "k_distribute.cu")
MARK = [("// ---- A: load + encode", "A encode"), ("// ---- B: read starts", "B read starts"),
        ("// validity masks by doubling", "validity"), ("// ---- C: canonical p-mer keys", "C p-mer keys"),
        ("// ---- D: sliding minimum", "D/E sliding min"), ("// ---- F: super-k-mers", "F runs"),
        ("// G: records of the runs", "G emission"), ("// carry the rest", "carry"),
        ("// ---- per-warp statistics", "stats")]
lines = open(SRC).read().split("\n")
bounds = []
for m, name in MARK:
    for i, l in enumerate(lines):
        if m in l:
            bounds.append((i + 1, name))
            break
bounds.append((10**9, "end"))
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
