"""One-off parity stress: the EVD kernels (f64/f32, real/complex, all flags)
against the oracle on several seeds at 2^22 matrices each, and the batched SVD
on 4 seeds x 512 matrices.  Prints one summary line per case; exit 1 on any
mismatch.  usage: PYTHONPATH=. python scripts/stress_parity.py"""
import sys

import numpy as np
import torch

import oracle as O
import paper_2202_08361_b200 as J
import synth

bad = 0
r = 1 << 22
for seed in (101, 202, 303):
    for f32 in (False, True):
        for cplx in (False, True):
            gen = (synth.evd_cfg2_f32 if cplx else synth.evd_cfg1_f32) if f32 else \
                (synth.evd_cfg2 if cplx else synth.evd_cfg1)
            a = gen(r, seed=seed)
            for flags in (0, 3):
                g = J.evd2_batched(*[torch.from_numpy(x).cuda() for x in a], flags=flags)
                torch.cuda.synchronize()
                ref = (O.evd2_batched_f32 if f32 else O.evd2_batched)(*a, flags=flags)
                u = np.uint32 if f32 else np.uint64
                ok = all(np.array_equal(g[k].cpu().numpy().view(u), ref[k].view(u))
                         for k in ("lam1", "lam2", "cos", "sin_re") + (("sin_im",) if cplx else ()))
                ok = ok and np.array_equal(g["zeta"].cpu().numpy(), ref["zeta"])
                ok = ok and np.array_equal(g["perm"].cpu().numpy().view(np.uint32), ref["perm"])
                print(f"evd seed={seed} f32={f32} cplx={cplx} flags={flags} r={r}: "
                      f"{'bitwise' if ok else 'MISMATCH'}", flush=True)
                bad += not ok
for seed in (11, 22, 33, 44):
    for cplx in (False, True):
        A = synth.svd_cfg4(512, seed=seed)
        if not cplx:
            A = np.ascontiguousarray(A.real)
        W, c, offs = J.batched_rspec(cplx, 64)
        ref = O.gesvj_batched(A, O.RSpec.make(W, c, offs), max_sweeps=30)
        g = torch.from_numpy(np.ascontiguousarray(np.transpose(A, (0, 2, 1)))).cuda().transpose(1, 2)
        out = J.gesvj_batched(g, max_sweeps=30)
        torch.cuda.synchronize()
        U = np.ascontiguousarray(out["U"].transpose(1, 2).contiguous().cpu().numpy().transpose(0, 2, 1))
        ok = np.array_equal(U.view(np.uint64), np.ascontiguousarray(ref["U"]).view(np.uint64))
        ok = ok and np.array_equal(out["sigma"].cpu().numpy().view(np.uint64),
                                   np.ascontiguousarray(ref["sigma"]).view(np.uint64))
        ok = ok and np.array_equal(out["sweeps"].cpu().numpy(), ref["sweeps"])
        print(f"batched seed={seed} cplx={cplx} 512 x 64x32: {'bitwise' if ok else 'MISMATCH'}",
              flush=True)
        bad += not ok
print("ALL BITWISE" if bad == 0 else f"{bad} MISMATCHES")
sys.exit(1 if bad else 0)
