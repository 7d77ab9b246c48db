"""Opcode histogram of the hottest loop of a kernel's SASS (the backward branch whose body
holds the most instructions of a given opcode, DSETP by default).

    cuobjdump -sass -fun <mangled> obj.o > k.sass && python tools/sass_loop.py k.sass [OPC]
"""
import collections
import re
import sys

LINE = re.compile(r"^\s+/\*([0-9a-f]{4,})\*/\s+(.*?);")


def parse(path):
    ins = []
    for ln in open(path):
        m = LINE.match(ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    return ins


def opcode(text):
    t = text
    if t.startswith("@"):
        t = t.split(None, 1)[1]
    return t.split()[0].split(".")[0]


def main():
    ins = parse(sys.argv[1])
    key = sys.argv[2] if len(sys.argv) > 2 else "DSETP"
    addr_idx = {a: k for k, (a, _) in enumerate(ins)}
    best = None
    for k, (a, t) in enumerate(ins):
        if opcode(t) != "BRA":
            continue
        m = re.search(r"0x([0-9a-f]+)", t.split("BRA", 1)[1])
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= a or tgt not in addr_idx:
            continue
        body = ins[addr_idx[tgt]:k + 1]
        n = sum(1 for _, x in body if opcode(x) == key)
        if best is None or n > best[0]:
            best = (n, tgt, a, body)
    if best is None:
        print("no loop")
        return
    n, tgt, a, body = best
    c = collections.Counter(opcode(x) for _, x in body)
    print(f"loop {tgt:#x}..{a:#x}: {len(body)} instructions, {n} {key}")
    for op, cnt in c.most_common():
        print(f"  {op:10s} {cnt}")


if __name__ == "__main__":
    main()
