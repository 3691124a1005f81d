"""Quick U1 tcgen05 probe run (scratch tool): int8 MAC/s per (M, N)."""
import ctypes, os, sys
lib = ctypes.CDLL(os.path.join(os.path.dirname(__file__), "..", "paper_2409_05205_b200", "libhe_u1.so"))
lib.u1_run.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p] * 3
import torch
torch.cuda.init()
names = {5: "mma.sync m16n8k32", 9: "tc M128 N16", 10: "tc M128 N32", 11: "tc M128 N64",
         12: "tc M128 N256", 13: "tc M64 N32", 14: "tc M64 N256"}
for w, n in names.items():
    ms, cyc, ops = ctypes.c_float(), ctypes.c_longlong(), ctypes.c_double()
    blocks, threads = (148 * 8, 256) if w == 5 else (148, 128)
    rc = lib.u1_run(w, blocks, threads, 2000 if w == 5 else 4000, ctypes.byref(ms), ctypes.byref(cyc), ctypes.byref(ops))
    rate = ops.value / (ms.value * 1e-3)
    print(f"{n:22s} rc={rc} {rate:.3e} MAC/s  {rate/148/1.965e9:.0f} MAC/clk/SM  ms={ms.value:.3f} cyc={cyc.value}")
