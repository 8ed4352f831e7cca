"""Per-kernel SASS opcode summary of libls_eval.so (cuobjdump -sass), for profiles/.

    python tools/sass_summary.py [paper_2509_00217_b200/libls_eval.so] > profiles/r02_sass_opcodes.txt

Counts static instructions per kernel and the mnemonics that show the design:
UBLKCP (TMA bulk copies), SYNCS.* (mbarrier), DADD/DMUL/DFMA/DSETP (fp64),
MUFU.RCP64H (fp64 division seeds), REDUX/VOTE/SHFL (warp reductions).
"""
import re
import subprocess
import sys
from collections import Counter

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2509_00217_b200/libls_eval.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
kernels, cur = {}, None
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        kernels[cur] = Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m and cur:
        kernels[cur][m.group(2)] += 1
KEYS = ("UBLKCP", "SYNCS", "DADD", "DMUL", "DFMA", "DSETP", "MUFU.RCP64H", "REDUX", "VOTE", "SHFL", "LDS", "STG",
        "LDG", "ATOMG", "RED")


def pick(c, key):
    return sum(v for k, v in c.items() if k == key or k.startswith(key + "."))


def short(name):
    dm = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    return dm.replace("(anonymous namespace)::", "").replace("ls::", "")[:110]


print(f"{'kernel':110s} {'instr':>7s} " + " ".join(f"{k.split('.')[0][:6]:>6s}" for k in KEYS))
for name, c in sorted(kernels.items(), key=lambda kv: -sum(kv[1].values())):
    if "eval_ws_kernel" not in name and "sweep_kernel" not in name and "valid_" not in name \
            and "eval_one" not in name and "sa_chain" not in name and "topk_merge_fast" not in name:
        continue
    print(f"{short(name):110s} {sum(c.values()):7d} " + " ".join(f"{pick(c, k):6d}" for k in KEYS))
