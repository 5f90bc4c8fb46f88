"""SASS instruction census of the hot kernels (cuobjdump -sass over the built
objects): tensor-core (DMMA, UTCIMMA = tcgen05.mma), TMA (UTMALDG, UBLKCP),
TMEM (LDTM), barrier and memory instruction counts per kernel.
  python tools/sass_census.py > profiles/sass_census_r02.json"""
import collections, json, re, subprocess, sys
from pathlib import Path
OBJ = Path(__file__).resolve().parents[1] / "paper_2110_02820_b200" / "build_obj"
KEEP = ("gemm_dmma_kernel", "pcg_persistent_kernel", "kfree_sym_kernel", "i8_gemm_kernel", "ozaki_split",
        "kblock_kernel")
OPS = ("DMMA", "UTCIMMA", "UTCBAR", "LDTM", "UTMALDG", "UBLKCP", "SYNCS", "DFMA", "DMUL", "DADD", "LDS", "LDG",
       "STG", "STS", "ATOMS", "BAR", "SHFL")
out = {}
for obj in sorted(OBJ.glob("*.o")):
    sass = subprocess.run(["cuobjdump", "-sass", str(obj)], capture_output=True, text=True).stdout
    name = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            name = m.group(1) if any(k in m.group(1) for k in KEEP) else None
            if name:
                out[name] = collections.Counter()
            continue
        if name is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            out[name]["instructions"] += 1
            op = m.group(1)
            for k in OPS:
                if op == k or op.startswith(k):
                    out[name][k] += 1
                    break
json.dump({k: dict(v) for k, v in out.items()}, sys.stdout, indent=1)
