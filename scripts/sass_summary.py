"""SASS evidence for the hot kernels: registers / stack / local memory (cuobjdump
-res-usage) and opcode counts (cuobjdump -sass) -- TMA bulk copies (UBLKCP),
mbarrier ops (SYNCS), MUFU.RSQ64H, REDG vs ATOMG, FP64 mix, spills (LDL/STL).

python scripts/sass_summary.py [lib.so] > profiles/rNN_sass_summary.json
"""
import collections
import json
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1502_03391_b200/libjofc_gpu.so"
KERNELS = {
    "jofc_pass_kernel<5>": "_ZN8jofc_gpu16jofc_pass_kernelILi5EEEvNS_10PassParamsE",
    "jofc_pass_kernel<3>": "_ZN8jofc_gpu16jofc_pass_kernelILi3EEEvNS_10PassParamsE",
    "jofc_solve_persistent_kernel<3>": "_ZN8jofc_gpu28jofc_solve_persistent_kernelILi3EEEvNS_10PassParamsE",
    "jofc_solve_persistent_kernel<2>": "_ZN8jofc_gpu28jofc_solve_persistent_kernelILi2EEEvNS_10PassParamsE",
    "jofc_epilogue_kernel<5>": "_ZN8jofc_gpu20jofc_epilogue_kernelILi5EEEvNS_9EpiParamsE",
    "jofc_epilogue_wide_kernel<5,256>": "_ZN8jofc_gpu25jofc_epilogue_wide_kernelILi5ELi256EEEvNS_9EpiParamsE",
    "jofc_epilogue_wide_kernel<3,1024>": "_ZN8jofc_gpu25jofc_epilogue_wide_kernelILi3ELi1024EEEvNS_9EpiParamsE",
    "jofc_oos_solve_kernel<3>": "_ZN8jofc_gpu21jofc_oos_solve_kernelILi3EEEvNS_10OospParamsE",
    "jofc_oos_step_kernel<3>": "_ZN8jofc_gpu20jofc_oos_step_kernelILi3EEEvNS_9OosParamsE",
    "jofc_oos_pass_kernel<3>": "_ZN8jofc_gpu20jofc_oos_pass_kernelILi3EEEvNS_9OosParamsE",
}
CLASSES = ["DFMA", "DADD", "DMUL", "MUFU", "UBLKCP", "SYNCS", "REDG", "ATOMG", "ATOMS", "LDS",
           "STS", "SHFL", "LDG", "STG", "LDL", "STL", "BAR", "MEMBAR", "FENCE"]


def res_usage():
    out = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    res, cur = {}, None
    for line in out.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", line)
        if m and cur:
            res[cur] = dict(zip(("registers", "stack", "shared_static", "local"),
                                map(int, m.groups())))
    return res


def opcodes(mangled):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", mangled, LIB], capture_output=True,
                         text=True).stdout
    cnt = collections.Counter()
    for line in out.splitlines():
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if not m:
            continue
        op = m.group(2)
        full = op
        base = op.split(".")[0]
        cnt[base] += 1
        if full.startswith("MUFU.RSQ64H"):
            cnt["MUFU.RSQ64H"] += 1
    return cnt


def main():
    res = res_usage()
    data = {}
    for name, mangled in KERNELS.items():
        c = opcodes(mangled)
        fp64 = c["DFMA"] + c["DADD"] + c["DMUL"]
        data[name] = {**res.get(mangled, {}),
                      "instructions": sum(v for k, v in c.items() if k != "MUFU.RSQ64H"),
                      "fp64_instructions": fp64,
                      "opcodes": {k: c[k] for k in CLASSES + ["MUFU.RSQ64H"] if c[k]}}
    print(json.dumps({"library": LIB, "tool": "cuobjdump -res-usage / -sass (CUDA 12.9)",
                      "note": "static counts over the whole kernel (both block-pair paths, "
                              "band / tail code); the C3 unmasked block body is 896 FP64 of "
                              "1068 instructions per 32 pairs (DESIGN.md section 4)",
                      "kernels": data}, indent=1))


if __name__ == "__main__":
    main()
