"""List the innermost loops of a cuobjdump -sass dump: body size, FFMA2-class count, local-memory ops."""
import re, sys
lines = open(sys.argv[1]).read().splitlines()
ins = []
for l in lines:
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
addr = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", t)
    if "BRA" in t:
        tgt = re.search(r"0x([0-9a-f]+)", t)
        if not tgt: continue
        ta = int(tgt.group(1), 16)
        if ta < a and ta in addr:
            body = [x[1] for x in ins[addr[ta]:i + 1]]
            n = len(body)
            if n > int(sys.argv[2] if len(sys.argv) > 2 else 400): continue
            c = lambda p: sum(1 for b in body if re.search(p, b))
            print(f"loop 0x{ta:x}-0x{a:x}: {n} instr, FP32x2 {c(r'F(FMA|MUL|ADD)2')}, FFMA/FMUL/FADD {c(r'\bF(FMA|MUL|ADD)\b')}, "
                  f"LDS {c(r'LDS')}, STS {c(r'STS')}, MUFU {c(r'MUFU')}, FMNMX {c(r'FMNMX')}, MOV {c(r'\bMOV')}, "
                  f"local {c(r'LDL|STL')}, SHFL {c(r'SHFL')}")
