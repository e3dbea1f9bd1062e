"""Static SASS loop census of one kernel: compile a device source to a cubin
for sm_100a and, for every backward branch, count the instructions of the
loop body by opcode (ALU / FMA-pipe split). Used to check an instruction
budget change before spending GPU time.

    python tools/sass_loops.py paper_1803_03288_b200/csrc/device/sweep.cu 'chain_sweep_kernelIhLb0EiLb0E'
"""
import collections
import os
import re
import subprocess
import sys

src, pat = sys.argv[1], sys.argv[2]
out = "/tmp/sass/" + os.path.basename(src) + ".cubin"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-O3", "-cubin",
                "--expt-relaxed-constexpr", "-Iinclude", "-o", out, src], check=True)
sass = subprocess.run(["cuobjdump", "-sass", out], capture_output=True, text=True, check=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)
ALU = {"LOP3", "SHF", "ISETP", "IADD3", "VIMNMX", "SEL", "LEA", "MOV", "VIADDMNMX", "PRMT", "FMNMX", "SGXT", "BMSK",
       "POPC", "FLO", "IABS", "LOP", "PLOP3", "P2R", "R2P"}
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ins = []
    for line in f.split("\n"):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    addr = {a: k for k, (a, _) in enumerate(ins)}
    print(name, len(ins), "instructions")
    for k, (a, txt) in enumerate(ins):
        m = re.search(r"BRA\s+(?:`?\(?\.L_x_\d+\)?|0x([0-9a-f]+))", txt)
        t = re.search(r"BRA\s+0x([0-9a-f]+)", txt)
        if not t:
            continue
        tgt = int(t.group(1), 16)
        if tgt >= a or tgt not in addr:
            continue
        body = ins[addr[tgt]:k + 1]
        if len(body) < 40:
            continue
        c = collections.Counter()
        for _, s in body:
            op = re.sub(r"^@!?U?P\w+\s+", "", s).split()[0].split(".")[0]
            c[op] += 1
        alu = sum(v for o, v in c.items() if o in ALU)
        fma = sum(v for o, v in c.items() if o in ("IMAD", "VIADD", "IADD", "FFMA", "HFMA2", "IMUL"))
        print(f"  loop {tgt:#x}..{a:#x}: {len(body)} inst  alu {alu}  fma {fma}  "
              + " ".join(f"{o}:{v}" for o, v in c.most_common(12)))
