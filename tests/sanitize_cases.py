"""Small searches through every kernel family, for compute-sanitizer runs:

compute-sanitizer --tool memcheck  python tests/sanitize_cases.py
compute-sanitizer --tool racecheck python tests/sanitize_cases.py

Covers the byte kernels (L_1 / L_marg / L_2, aligned and unaligned Algorithm-1 slices, the
grouped prefix hook; L_3 / L_4 with 1, 2 and 3 paired rows; the all-H L_3 kernel with 3 and 4),
the 16-bit and int32 families (LNORM_KERNEL), the generic kernel (also batched), the reductions,
the batched API (byte walks, 16-bit paired walk, generic kernel) and the device-input path (guard-statistics kernel, caller stream).  Every value is checked
against the oracle so a silent corruption also fails.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2503_21596_b200 as L  # noqa: E402
from paper_2503_21596_b200 import synth  # noqa: E402


def check(M, d=1, marg=False):
    v, _ = L.compute(M, d=d, with_marginals=marg)
    assert v == oracle.norm(M, d=d, with_marginals=marg)[0], (M.shape, d, marg)
    return L.last_stats()["variant"]


def main():
    seen = set()
    for n, m in [(12, 13), (13, 40), (11, 90)]:
        for d, marg in [(1, False), (1, True), (2, False)]:
            seen.add(check(synth.random_matrix(n, m, 500 + n + m), d, marg))
    M = synth.random_matrix(14, 16, 501)
    for sl in (3, 8):
        assert L.compute_sliced(M, sl)[0] == oracle.l1(M)[0]
    P = np.zeros((8, 9), dtype=np.int8)
    g = synth.SplitMix64(502)
    for i in range(8):
        P[i, 1:7] = [g.next() % 2 for _ in range(6)]
        P[i, :7] = P[i - i % 4, :7]
        P[i, 7], P[i, 8] = (i % 4) >> 1, (i % 4) & 1
    got = L.prefix_maxima(M, P)
    assert all(got[i] == oracle.prefix_max(M, P[i])[0] for i in range(8))
    for d in (3, 4):
        for n in (8, 10, 12, 14):
            seen.add(check(synth.random_matrix(n, 14, 510 + n + d), d))
    # L_3 all-H kernel with 3 and 4 paired rows, and past 32 columns; the all-E kernel
    for n, m in [(13, 14), (12, 40)]:
        seen.add(check(synth.random_matrix(n, m, 515 + n + m), 3))
    os.environ["LNORM_LDU8W"] = "0"
    seen.add(check(synth.random_matrix(13, 14, 516), 3))
    os.environ["LNORM_LDU8W"] = "1"
    for fam in ("pair16", "packed", "int32", "generic"):
        os.environ["LNORM_KERNEL"] = fam
        for d, marg in [(1, False), (1, True), (2, False), (3, False)]:
            seen.add(check(synth.random_matrix(11, 12, 520 + d), d, marg))
    os.environ["LNORM_KERNEL"] = "auto"
    R = np.array(synth.random_matrix(12, 14, 530), dtype=np.int64)
    R[5] = 2 * R[4]
    R[:, 3] = 0
    v, arg, _ = L.compute_reduced(R.astype(np.int32))
    assert v == oracle.l1(R.astype(np.int32))[0]
    Ms = np.stack([synth.random_matrix(10, 10, 540 + i) for i in range(16)])
    vals, _ = L.compute_batch(Ms)
    assert all(int(vals[i]) == oracle.l1(Ms[i])[0] for i in range(16))
    for d, n, m, b in ((1, 14, 16, 9), (2, 12, 12, 7), (3, 11, 14, 6), (3, 14, 23, 3), (4, 9, 10, 5)):   # batched byte walks
        Bs = np.stack([synth.random_matrix(n, m, 545 + 13 * i + d) for i in range(b)])
        vals, _ = L.compute_batch(Bs, d=d)
        seen.add(L.last_stats()["variant"])
        assert all(int(vals[i]) == oracle.norm(Bs[i], d=d)[0] for i in range(b))
    Ts = np.stack([synth.random_matrix(4, 3, 550 + i, -1, 1) for i in range(40)])     # generic batched walk
    for d in (1, 3):
        vals, _ = L.compute_batch(Ts, d=d)
        assert all(int(vals[i]) == oracle.norm(Ts[i], d=d)[0] for i in range(40))
    import torch                                                                  # device input + stream
    Md = torch.from_numpy(synth.random_matrix(12, 13, 560)).cuda()
    assert L.compute_device(Md, stream=torch.cuda.Stream())[0] == oracle.l1(Md.cpu().numpy())[0]
    print("sanitize cases ok; kernel variants:", sorted(L.VARIANTS[v] for v in seen))


if __name__ == "__main__":
    main()
