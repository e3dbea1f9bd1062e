"""Hot-path length of the shuffle loops: for each loop (backward branch), the
instructions on the fall-through path when every forward conditional branch
is assumed not taken except the unconditional ones (the rejection path is the
taken side of the first conditional branch in draw_group).

    python tools/sass_hot.py /tmp/sass/sweep.cu.cubin 'chain_sweep_kernelIhLb0EiLb0E'
"""
import re
import subprocess
import sys

cub, pat = sys.argv[1], sys.argv[2]
ALU = {"LOP3", "SHF", "ISETP", "IADD3", "VIMNMX", "SEL", "LEA", "MOV", "VIADDMNMX", "PRMT", "FMNMX", "SGXT", "BMSK",
       "POPC", "FLO", "IABS", "PLOP3", "P2R", "R2P"}
FMA = {"IMAD", "VIADD", "FFMA", "HFMA2", "IMUL"}
sass = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True, check=True).stdout
for f in re.split(r"\n\s*Function : ", sass)[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ins = []
    for line in f.split("\n"):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    idx = {a: k for k, (a, _) in enumerate(ins)}
    for k, (a, t) in enumerate(ins):
        m = re.search(r"BRA\s+0x([0-9a-f]+)", t)
        if not m or int(m.group(1), 16) >= a:
            continue
        start = idx.get(int(m.group(1), 16))
        if start is None or k - start < 60:
            continue
        # walk: conditional forward branches not taken, unconditional taken
        n, pc, seen = 0, start, set()
        alu = fma = 0
        while pc <= k and pc not in seen:
            seen.add(pc)
            n += 1
            t2 = ins[pc][1]
            op = re.sub(r"^@!?U?P\w+\s+", "", t2).split()[0].split(".")[0]
            alu += op in ALU
            fma += op in FMA
            mb = re.search(r"BRA\s+0x([0-9a-f]+)", t2)
            if mb and not t2.startswith("@") and pc != k:
                pc = idx[int(mb.group(1), 16)]
                continue
            pc += 1
        print(f"loop {ins[start][0]:#x}..{a:#x}: hot path {n} instructions (alu {alu}, fma {fma})")
