"""Which reduction placement is right on the mode-parity test shapes (debug)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import _lib, shard  # noqa: E402

dev = torch.device("cuda", 0)
MM = "(i,k),(k,j)->(i,j)"
for world in (1, 2):
    for splits in (None, 1, 3):
        for with_c0 in (False, True):
            M, N, K = 640, 384, 6144 + 64 * world
            g = torch.Generator(device=dev).manual_seed(world * 7 + (splits or 0))
            a = torch.randn(M, K, device=dev, generator=g).bfloat16()
            b = torch.randn(K, N, device=dev, generator=g).bfloat16()
            c0 = torch.randn(M, N, device=dev, generator=g).bfloat16() if with_c0 else None
            ks = [shard.k_range(K, world, r) for r in range(world)]
            A = [a[:, lo:hi] for lo, hi in ks]
            B = [b[lo:hi] for lo, hi in ks]
            want = a.double() @ b.double() + (c0.double() if with_c0 else 0)
            res = []
            for m in (_lib.RS_IN_KERNEL, _lib.RS_DEFERRED):
                o = shard.emulate_fused_ksplit(MM, A, B, c0=c0, mode=m, local_splits=splits)
                err = (o.double() - want).norm(dim=1) / want.norm(dim=1)
                bad = (err > 1e-2).nonzero().flatten().tolist()
                res.append((float((o.double() - want).norm() / want.norm()), bad[:3], len(bad)))
            print(world, splits, with_c0, res, flush=True)
