"""Per-kernel SASS statistics for liblorenz.so (run here, no GPU needed).

For each kernel: instruction count, FP64 opcode counts, local-memory traffic, and the
hottest loop (the backward branch target whose body holds the most DADD/DMUL),
reporting its DADD/DMUL/DFMA mix — the canonical RK4 step must be 43 DADD + 32 DMUL
and 0 DFMA.

Usage: python tools/sass_stats.py [path/to/liblorenz.so]
"""
import collections
import json
import re
import subprocess
import sys


def kernels(sass: str):
    cur, body = None, []
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
        elif cur:
            body.append(line)
    if cur:
        yield cur, body


INSN = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)")


def parse(body):
    out = []
    for ln in body:
        m = INSN.search(ln)
        if m:
            out.append((int(m.group(1), 16), m.group(3), ln))
    return out


def loop_stats(ins):
    best = None
    for addr, op, ln in ins:
        if op.startswith("BRA"):
            m = re.search(r"0x([0-9a-f]+)", ln.split("BRA", 1)[1])
            if not m:
                continue
            tgt = int(m.group(1), 16)
            if tgt < addr:
                ops = collections.Counter(o.split(".")[0] for a, o, _ in ins if tgt <= a <= addr)
                fp = ops["DADD"] + ops["DMUL"] + ops["DFMA"]
                score = fp / max(1, sum(ops.values())) if fp >= 10 else 0.0  # densest FP64 loop
                if best is None or score > best[0]:
                    best = (score, tgt, addr, addr - tgt, ops)
    return best


def back_edges(ins):
    """(target, branch address) of every backward branch: the loops of the function."""
    out = []
    for addr, op, ln in ins:
        if op.startswith("BRA"):
            m = re.search(r"0x([0-9a-f]+)", ln.split("BRA", 1)[1])
            if m and int(m.group(1), 16) < addr:
                out.append((int(m.group(1), 16), addr))
    return out


def innermost_fp64_loops(ins, min_fp64=10):
    """Opcode counts of every innermost loop (no other loop inside it) with at least `min_fp64`
    DADD/DMUL/DFMA and no MUFU (a correctly rounded division's loop is not an integrator)."""
    edges = back_edges(ins)
    inner = [e for e in edges if not any(o != e and e[0] <= o[0] and o[1] <= e[1] for o in edges)]
    out = []
    for t, a in inner:
        c = collections.Counter(o.split(".")[0] for ad, o, _ in ins if t <= ad <= a)
        if c["DADD"] + c["DMUL"] + c["DFMA"] >= min_fp64 and not c["MUFU"]:
            out.append({"DADD": c["DADD"], "DMUL": c["DMUL"], "DFMA": c["DFMA"],
                        "other": sum(c.values()) - c["DADD"] - c["DMUL"] - c["DFMA"],
                        "other_ops": sorted({o for o in c if o not in ("DADD", "DMUL", "DFMA")})})
    return out


CHAIN = re.compile(r"(lorenz_chain(?:_seg)?_kernel)ILi(\d)ELi(\d)ELi(\d+)E")


def chain_kernel_loops(so):
    """{(kernel, OP, INTEG, CTA): ([innermost FP64 loops], local-memory instructions)} for every
    chain kernel instantiation in the library (cuobjdump -sass of those functions only)."""
    names = subprocess.run(["cuobjdump", "-res-usage", so], capture_output=True, text=True, check=True).stdout
    funs = sorted(set(re.findall(r"Function (_ZN2lz\w*lorenz_chain\w+):", names)))
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", ",".join(funs), so], capture_output=True, text=True,
                          check=True).stdout
    out = {}
    for name, body in kernels(sass):
        m = CHAIN.search(name)
        if not m:
            continue
        ins = parse(body)
        ops = collections.Counter(o.split(".")[0] for _, o, _ in ins)
        out[(m.group(1), int(m.group(2)), int(m.group(3)), int(m.group(4)))] = (
            innermost_fp64_loops(ins), ops["LDL"] + ops["STL"])
    return out


def main():
    so = sys.argv[1] if len(sys.argv) > 1 else "paper_1201_3114_b200/csrc/liblorenz.so"
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
    report = {}
    for name, body in kernels(sass):
        ins = parse(body)
        ops = collections.Counter(o.split(".")[0] for _, o, _ in ins)
        best = loop_stats(ins)
        rep = {"instructions": len(ins), "DADD": ops["DADD"], "DMUL": ops["DMUL"], "DFMA": ops["DFMA"],
               "local_mem": ops["LDL"] + ops["STL"]}
        if best:
            lops = best[4]
            rep["hot_loop"] = {"instructions": sum(lops.values()), "DADD": lops["DADD"], "DMUL": lops["DMUL"],
                               "DFMA": lops["DFMA"],
                               "other": sum(lops.values()) - lops["DADD"] - lops["DMUL"] - lops["DFMA"]}
        report[name] = rep
    print(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
