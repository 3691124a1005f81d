"""One size's forward + inverse NTT through the C-ABI (for ncu captures):
python scripts/ntt_one.py N [limbs]."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2409_05205_b200 as he  # noqa: E402

N = int(sys.argv[1])
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 256
primes = {8192: synth.PRIMES_N8192[:2], 16384: synth.PRIMES_N16384[:2],
          32768: synth.PRIMES_N32768[:2]}[N]
ctx = he.Context(list(primes), N.bit_length() - 1, 65537, 0)
buf = torch.from_numpy(synth.uniform_residues((nl // 2, 2, N), list(primes), 7, "misc", N)
                       .view(np.int64)).cuda()
for _ in range(2):
    ctx.ntt_forward(buf)
    ctx.ntt_inverse(buf)
torch.cuda.synchronize()
print("ok")
