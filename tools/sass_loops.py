"""List the loops (backward branches) of one kernel in a cuobjdump -sass dump
with their instruction mix: python tools/sass_loops.py dump.sass KERNEL_REGEX"""
import collections
import re
import sys

text = open(sys.argv[1]).read()
pat = re.compile(sys.argv[2])
funcs = re.split(r"\n\s*Function : ", text)
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    if not pat.search(name):
        continue
    ins = []
    for m in re.finditer(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", f):
        ins.append((int(m.group(1), 16), m.group(2).strip()))
    addr = {a: i for i, (a, _) in enumerate(ins)}
    print(name[:110])
    for i, (a, s) in enumerate(ins):
        m = re.search(r"BRA\S*\s+(?:P\d, |!?U?P\d, )?0x([0-9a-f]+)", s)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < a and tgt in addr and i - addr[tgt] > 20:
                body = [x for _, x in ins[addr[tgt]:i + 1]]
                ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", x).split()[0].split(".")[0] for x in body)
                n2 = ops["FFMA2"] + ops["FADD2"] + ops["FMUL2"]
                print(f"  loop {tgt:#x}-{a:#x}: {len(body)} instr, FP2={n2}, MUFU={ops['MUFU']}, "
                      + ", ".join(f"{k}={v}" for k, v in ops.most_common(12)))
