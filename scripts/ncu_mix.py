"""Developer tool: executed warp-instruction mix per opcode / pipe of the kernel in an .ncu-rep (source page)."""
import csv, subprocess, sys, io, collections
rep = sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]; data = rows[2:]
ia, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
FMA = {"IMAD", "FFMA", "FMUL", "FADD", "IDP", "HFMA2", "IMAD.MOV", "IMAD.SHL", "IMAD.WIDE", "IMAD.IADD", "IMAD.HI", "IMAD.X", "HADD2", "FSEL"}
ALU = {"IADD3", "LOP3", "SHF", "PRMT", "ISETP", "SEL", "MOV", "IABS", "LEA", "POPC", "FLO", "BREV", "VIADD", "VIMNMX", "IMNMX", "SGXT", "BMSK", "PLOP3", "CS2R", "LOP", "IADD", "R2P", "P2R", "FMNMX", "VABSDIFF", "VIADDMNMX", "IADD.64", "UIADD3"}
LSU = {"LDS", "STS", "LDG", "STG", "ATOMS", "ATOMG", "RED", "LDGSTS", "LDSM", "LD", "ST", "ATOM", "LDC", "LDL", "STL", "REDG"}
ops = collections.Counter(); pipes = collections.Counter()
tot = 0
for r in data:
    c = int(r[ia]); s = r[isrc].strip()
    if not c or not s: continue
    parts = s.split()
    op = parts[1] if parts[0].startswith("@") else parts[0]
    base = op.split(".")[0]
    ops[op if base in ("IMAD",) else base] += c
    tot += c
    if base in FMA: pipes["fma"] += c
    elif base in ALU: pipes["alu"] += c
    elif base in LSU: pipes["lsu"] += c
    elif base in ("SHFL", "VOTE", "MATCH", "REDUX", "WARPSYNC", "BAR", "BSSY", "BSYNC", "BRA", "EXIT", "NOP", "YIELD", "CALL", "RET", "DEPBAR", "ERRBAR", "MEMBAR", "S2R", "S2UR", "NANOSLEEP", "BREAK", "BRX", "JMP"): pipes["ctl/other:" + base] += c
    elif base.startswith("U") or base in ("R2UR", "UMOV"): pipes["uniform"] += c
    else: pipes["?" + base] += c
print(f"total {tot/1e6:.1f}M")
for k, v in pipes.most_common(): print(f"  {k:22s} {v/1e6:8.1f}M {100*v/tot:5.1f}%")
print("top opcodes:")
for k, v in ops.most_common(40): print(f"  {k:22s} {v/1e6:8.1f}M {100*v/tot:5.1f}%")
