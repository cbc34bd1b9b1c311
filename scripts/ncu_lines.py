"""Debug: executed warp-instructions per source line (top N) of each kernel in an ncu report
captured with --import-source on.  Usage: python scripts/ncu_lines.py report.ncu-rep [top] [per]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
per = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
kern = None; f = None; hdr = None; res = {}
for r in csv.reader(io.StringIO(raw)):
    if len(r) < 2: continue
    if r[0] == "Kernel Name": kern = r[1][:60]; continue
    if r[0] == "Function Name": kern = r[1][:60]; continue
    if r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; ie = hdr.index("Instructions Executed"); ss = hdr.index("Warp Stall Sampling (All Samples)"); continue
    if hdr and len(r) > ie and r[0] != "" and r[2] == "-":
        try: n = int(r[ie]); s = int(r[ss])
        except ValueError: continue
        res.setdefault(kern, []).append((n, s, f, int(r[0]), r[1].strip()[:80]))
for k, v in res.items():
    tot = sum(x[0] for x in v); st = sum(x[1] for x in v)
    print(f"== {k}: {tot} warp-instr, {st} stall samples")
    for x in sorted(v, reverse=True)[:top]:
        print(f"  {x[0] / per:10.1f} {x[1]:5d}  {x[2]}:{x[3]}  {x[4]}")
