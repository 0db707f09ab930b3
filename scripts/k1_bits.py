"""Dump K1 outputs (conf / argmax bits) for a fixed set of seeded inputs, so two library variants
(LOPA_LIB_VARIANT) can be compared bit for bit.  Both K1 forms use the same canonical slices and
folds, so their outputs must be identical.

    LOPA_LIB_VARIANT=ldg python scripts/k1_bits.py out_ldg.npz
    python scripts/k1_bits.py --compare out_base.npz out_ldg.npz
"""
import sys

import numpy as np


def main():
    if sys.argv[1] == "--compare":
        a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
        bad = 0
        for key in a.files:
            if not np.array_equal(a[key].view(np.uint32), b[key].view(np.uint32)):
                n = int((a[key].view(np.uint32) != b[key].view(np.uint32)).sum())
                print(f"MISMATCH {key}: {n} elements")
                bad += 1
        print(f"compared {len(a.files)} arrays: {'IDENTICAL' if not bad else f'{bad} differ'}")
        sys.exit(1 if bad else 0)
    import torch
    sys.path.insert(0, ".")
    from paper_2512_16229_b200 import lopa
    dev = torch.device("cuda:0")
    g = torch.Generator(device="cpu").manual_seed(1234)
    out = {}
    cases = [(151936, 241, 0), (151936, 256, 1), (64, 24, 0), (1000, 300, 0), (8193, 37, 1),
             (16391, 5, 0), (151936, 3, 0), (131075, 600, 1), (7, 1000, 0), (1 << 20, 9, 0)]
    for ci, (V, R, masked) in enumerate(cases):
        ld = (V + 7) // 8 * 8
        x = (torch.randn((R, ld), generator=g) * 3).to(torch.bfloat16)
        if R > 2:
            x[1, :] = float("-inf")
            x[1, min(5, V - 1)] = 4.0
            x[2, :V] = 1.0  # flat row: ties everywhere, argmax 0
        x = x.to(dev)
        mask = None
        if masked:
            mask = (torch.rand((R,), generator=g) < 0.6).to(torch.uint8).to(dev)
        conf, amax, st = lopa.confidence(x, vocab=V, row_mask=mask)
        torch.cuda.synchronize()
        c = conf.cpu().numpy()
        a = amax.cpu().numpy()
        if mask is not None:
            m = mask.cpu().numpy().astype(bool)
            c = np.where(m, c, 0).astype(np.float32)
            a = np.where(m, a, 0).astype(np.int32)
        out[f"conf{ci}"] = c
        out[f"amax{ci}"] = a
    np.savez(sys.argv[1], **out)
    print("wrote", sys.argv[1], len(out))


if __name__ == "__main__":
    main()
