import csv, io, subprocess, sys, collections
rep = sys.argv[1]
# an .ncu-rep, or the csv of `ncu -i REP --page source --csv --print-source sass`
out = (open(rep).read() if rep.endswith(".csv") else
       subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout)
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]; ie = h.index("Instructions Executed"); src = h.index("Source"); st=h.index("Warp Stall Sampling (All Samples)")
ops = collections.Counter(); stalls=collections.Counter(); tot=0; stot=0
for r in rows[1:]:
    try: n = int(r[ie])
    except: continue
    op = r[src].split()[0] if r[src].split() else "?"
    if op.startswith("@"): op = r[src].split()[1]
    op = op.split(".")[0]
    ops[op]+=n; tot+=n
    s=int(r[st] or 0); stalls[op]+=s; stot+=s
print("total warp instr", tot)
for op,n in ops.most_common(30): print(f"{op:10s} {n:12d} {n/tot:6.1%}  stall-samples {stalls[op]/max(stot,1):6.1%}")
