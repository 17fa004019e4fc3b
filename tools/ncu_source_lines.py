"""Aggregate an ncu report's source page per CUDA line: share of executed warp instructions and
of stall samples.  Usage: python tools/ncu_source_lines.py report.ncu-rep [top]"""
import csv, sys, subprocess, io
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
fname = None; hdr = None; out = []
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr and r[0].isdigit() and len(r) == len(hdr):
        ie = r[hdr.index("Instructions Executed")]
        ss = r[hdr.index("Warp Stall Sampling (All Samples)")]
        if ie not in ("-", "", "0"):
            out.append((int(ie), int(ss) if ss.isdigit() else 0, fname, int(r[0]), r[1][:110]))
tot = sum(o[0] for o in out); tots = sum(o[1] for o in out)
print("total warp instr", tot, "samples", tots)
for o in sorted(out, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*o[0]/tot:5.1f}% {100*o[1]/max(tots,1):5.1f}%  {o[2]}:{o[3]}  {o[4]}")
