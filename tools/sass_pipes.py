"""Static instruction mix of one kernel (by SASS opcode and by the pipe it issues to).

Usage: python tools/sass_pipes.py <kernel-substring> [lib.so] [--range START END]
Pipes (Blackwell, per B300_MICROARCH.md and ncu pipe names): alu = LOP3/ISETP/IADD3/
SHF/PRMT/FMNMX/SEL/...; fmaheavy = IMAD*/IDP; fma = FMUL/FFMA/FADD (either half);
xu = F2I/I2F/MUFU/FRND; lsu = LDG/STG/LDS/STS/SHFL/ATOM/RED.
"""
import re, subprocess, sys, collections, os

PIPE = {
    "LOP3": "alu", "ISETP": "alu", "FSETP": "alu", "IADD3": "alu", "SHF": "alu", "PRMT": "alu",
    "FMNMX": "alu", "VIMNMX": "alu", "VIMNMX3": "alu", "SEL": "alu", "FSEL": "alu", "LEA": "alu",
    "MOV": "alu", "PLOP3": "alu", "IABS": "alu", "BMSK": "alu", "FLO": "alu", "POPC": "alu",
    "ISCADD": "alu", "IMNMX": "alu", "P2R": "alu", "R2P": "alu", "LOP": "alu", "SGXT": "alu", "FCHK": "alu",
    "IMAD": "fmaheavy", "IDP": "fmaheavy", "IMUL": "fmaheavy", "IMMA": "tensor",
    "FMUL": "fma", "FFMA": "fma", "FADD": "fma", "FMUL2": "fma", "FADD2": "fma", "FFMA2": "fma", "VIADD": "fma?",
    "F2I": "xu", "I2F": "xu", "MUFU": "xu", "FRND": "xu", "F2F": "xu", "I2I": "xu", "F2FP": "alu",
    "LDG": "lsu", "STG": "lsu", "LDS": "lsu", "STS": "lsu", "SHFL": "lsu", "ATOMG": "lsu", "RED": "lsu",
    "REDG": "lsu", "ATOMS": "lsu", "LD": "lsu", "ST": "lsu", "LDC": "lsu",
}


def main():
    name = sys.argv[1]
    lib = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else \
        os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2306_11987_b200", "libint4linear.so")
    rng = None
    if "--range" in sys.argv:
        i = sys.argv.index("--range")
        rng = (int(sys.argv[i + 1], 16), int(sys.argv[i + 2], 16))
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", out)
    for f in funcs[1:]:
        fname = f.split("\n", 1)[0].strip()
        if name not in fname:
            continue
        ops, pipes = collections.Counter(), collections.Counter()
        n = 0
        for m in re.finditer(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)((?:\.[A-Z0-9_]+)*)", f):
            addr = int(m.group(1), 16)
            if rng and not (rng[0] <= addr < rng[1]):
                continue
            op = m.group(3)
            full = op + m.group(4)
            if op in ("NOP",):
                continue
            ops[full] += 1
            p = PIPE.get(op, "other")
            if op == "IMAD" and ".WIDE" in m.group(4):
                p = "fmaheavy"
            pipes[p] += 1
            n += 1
        print(f"== {fname}: {n} instructions")
        print("   pipes:", dict(pipes.most_common()))
        print("   ops:  ", ", ".join(f"{k}:{v}" for k, v in ops.most_common(40)))


if __name__ == "__main__":
    main()
