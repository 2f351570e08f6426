"""FP64 peak and latency microbenchmarks (libjofc_probe.so) on cuda:0."""
import ctypes as C
import os

lib = C.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                          "paper_1502_03391_b200", "libjofc_probe.so"))
a, b, c, d = (C.c_double() for _ in range(4))
lib.jofc_probe_fp64(0, C.byref(a), C.byref(b), C.byref(c))
print(f"DFMA {a.value:.2f} TF/s  DMMA {b.value:.2f} TF/s  DFMA+DMMA {c.value:.2f} TF/s")
lib.jofc_probe_latency(0, C.byref(a), C.byref(b), C.byref(c), C.byref(d))
print(f"latency cycles: DFMA {a.value:.1f}  DADD {b.value:.1f}  RSQ64H+DADD {c.value:.1f}  "
      f"SHFL.64+DADD {d.value:.1f}")
t = C.c_double()
for w in (4, 8, 12, 16, 32):
    row = []
    for ch in (1, 2, 4, 8, 16):
        lib.jofc_probe_occupancy(0, w, ch, C.byref(t))
        row.append(f"{t.value:6.2f}")
    print(f"warps/SM {w:2d}: chains 1,2,4,8,16 -> " + " ".join(row) + " TF/s")
gp, regs = C.c_double(), C.c_int()
names = {0: "full", 1: "no col acc", 2: "no fid", 3: "no col, no fid", 4: "fp32 seed",
         8: "shared product", 12: "shared product + fp32 seed", 16: "magic + 2 fp32 Newton seed"}
for d in (5, 3):
    for g in (1, 4):
        for fl in (0, 16):
            lib.jofc_probe_pair_math(0, d, g, fl, C.byref(gp), C.byref(regs))
            print(f"pair math d={d} G={g} {names[fl]:28s}: {gp.value:7.1f} Gpairs/s ({regs.value} regs)"
                  f" C3-equiv pass {4e8 / (gp.value * 1e9) * 1e3:.3f} ms")
pc = C.c_double()
for op, name in ((0, "MUFU.RSQ64H"), (1, "MUFU.RSQ f32"), (2, "DADD"), (3, "DMUL"),
                 (4, "DFMA 3 regs"), (5, "DFMA 1 reg"), (6, "DFMA acc form"),
                 (7, "DADD 2 regs"), (8, "7 DFMA + 1 RSQ64H"), (9, "8 DFMA + select"),
                 (10, "F2F.F32.F64+DMUL"), (11, "7 DFMA + F2F,RSQf32,F2F")):
    lib.jofc_probe_op(0, op, C.byref(pc))
    print(f"{name:13s}: {pc.value:.3f} warp-instr/clk/SM (at max clock)")
me = C.c_double()
lib.jofc_probe_rsq_error(0, C.byref(me))
import math
print(f"MUFU.RSQ64H seed: max |1 - s y0^2| = {me.value:.3e} (2^{math.log2(me.value):.2f}); "
      f"2nd-order error ~ 3e^2/8 = {3 * me.value**2 / 8:.2e}, 3rd-order ~ 5e^3/16 = "
      f"{5 * me.value**3 / 16:.2e}")
