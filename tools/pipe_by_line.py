"""FMA-heavy / ALU pipe load by CUDA source line from an ncu source-page export:
  ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass -k regex:KERNEL > src.csv
  python tools/pipe_by_line.py src.csv
Executed SASS instructions are weighted by the pipe cycles they cost on sm_100 (measured against
sm__pipe_fmaheavy_cycles_active: IMAD.WIDE 4 FMA-heavy cycles per warp instruction, IMAD/VIADD 2;
IADD3/LOP3/SHF/SEL/LEA/ISETP/MOV/PRMT 2 ALU cycles)."""
import csv,sys,re,collections
rows=list(csv.reader(open(sys.argv[1])))
fn=None; line=None; src=None
cost=collections.Counter(); inst=collections.Counter(); alu=collections.Counter(); srcs={}
W={'IMAD.WIDE':4,'IMAD.WIDE.U32':4,'IMAD.WIDE.U32.X':4,'IMAD.WIDE.X':4}
ALU=('IADD3','LOP3','SHF','SEL','LEA','ISETP','MOV','PRMT','FLO','POPC','IABS','IMNMX','VIMNMX')
tot_h=0;tot_i=0;tot_a=0
for r in rows:
    if not r: continue
    if r[0]=='File Path': fn=r[1].split('/')[-1]; continue
    if len(r)<8 or r[0] in ('Line No','Function Name'): continue
    if r[0]!='':
        line=f"{fn}:{r[0]}"; srcs[line]=r[1][:90]; continue
    s=r[3].strip()
    m=re.match(r'(@!?U?P\w+\s+)?([A-Z0-9_.]+)',s)
    if not m: continue
    op=m.group(2)
    try: n=int(r[7].replace(',',''))
    except: continue
    base=op.split('.')[0]
    h=0
    if op in W: h=4
    elif base in ('IMAD','VIADD','IMUL'): h=2
    a=2 if base in ALU else 0
    cost[line]+=h*n; inst[line]+=n; alu[line]+=a*n
    tot_h+=h*n; tot_i+=n; tot_a+=a*n
print("total warp instr",tot_i,"heavy cycles",tot_h,"alu cycles",tot_a)
for l,c in cost.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{c/tot_h*100:5.1f}% heavy {inst[l]/tot_i*100:5.1f}% inst {alu[l]/tot_a*100:5.1f}% alu  {l}  {srcs.get(l,'')}")
