#!/usr/bin/env python
"""Shared-memory bank model of the 3D Q2 (K = 2) contraction stages of force_kernel (no GPU).

Wavefronts of one warp-wide shared access: 64-bit accesses run as two half-warp phases,
128-bit ones as four quarter-warp phases; a phase costs the largest number of distinct
4-byte words that fall into one of the 32 banks.  Calibrated against ncu's per-line
"L1 Wavefronts Shared" of profiles/r02_q2_c4_force_full (stage-1 stores 56, stage-2 loads 54,
stage-2 stores 108, b2 loads 54, b3 loads 28 per unit: all reproduced).

    python tools/bank_sim.py        # Q2: the round-1 layout vs LAYOUT_K2 = 1;
                                    # Q3: the stage-2 task order without / with PERM_K3
"""
from collections import defaultdict

N, Q, NF, DIM, NT = 3, 4, 2, 3, 64


def _phase(addrs, size):
    banks = defaultdict(set)
    for a in addrs:
        if a is None:
            continue
        for w in range(size // 4):
            word = a // 4 + w
            banks[word % 32].add(word)
    return max((len(v) for v in banks.values()), default=0)


def warp_wavefronts(addrs, size):
    ph = {4: 1, 8: 2, 16: 4}[size]
    n = 32 // ph
    return sum(_phase(addrs[i * n:(i + 1) * n], size) for i in range(ph))


def cost(T, addr_fns, size=8):
    """T tasks over NT threads (rounds of NT); addr_fns: task -> double index, one per access"""
    tot = 0
    for t0 in range(0, T, NT):
        for af in addr_fns:
            for w in range(NT // 32):
                ad = []
                for l in range(32):
                    t = t0 + w * 32 + l
                    ad.append(8 * af(t) if t < T else None)
                tot += warp_wavefronts(ad, size)
    return tot


def forward(SFC, SBG, S1Q1, S2FC, S2K, S2Q1, order2):
    T1 = NF * DIM * N * N
    dec1 = lambda t: (t // (N * N), (t % (N * N)) % N, (t % (N * N)) // N)   # fc, a2, a3
    st1 = [lambda t, bg=bg, q1=q1: (lambda fc, a2, a3: fc * SFC + bg * SBG + q1 * S1Q1 + a3 * N + a2)(*dec1(t))
           for bg in range(2) for q1 in range(Q)]
    T2 = NF * DIM * Q * N

    def dec2(t):
        if order2 == "a3":
            return t // (Q * N), (t // N) % Q, t % N          # fc, q1, a3
        return t // (Q * N), t % Q, (t // Q) % N
    ld2 = [lambda t, bg=bg, a2=a2: (lambda fc, q1, a3: fc * SFC + bg * SBG + q1 * S1Q1 + a3 * N + a2)(*dec2(t))
           for bg in range(2) for a2 in range(N)]
    st2 = [lambda t, k=k, q2=q2: (lambda fc, q1, a3: fc * S2FC + k * S2K + q1 * S2Q1 + q2 * N + a3)(*dec2(t))
           for k in range(3) for q2 in range(Q)]
    fp = [lambda t, fc=fc, k=k, a3=a3: fc * S2FC + k * S2K + (t % 4) * S2Q1 + ((t // 4) % 4) * N + a3
          for fc in range(NF * DIM) for k in range(3) for a3 in range(N)]
    return dict(stage1_st=cost(T1, st1), stage2_ld=cost(T2, ld2), stage2_st=cost(T2, st2), fwd_point_ld=cost(64, fp))


def backward(TDL, TC, TQ1, TA3, WW, WC, WA, b2_q1fast=False):
    d1 = lambda t: (t // 16, (t % 16) % 4, (t % 16) // 4)                     # c, q1, q2
    b1s = [lambda t, dl=dl, a3=a3: (lambda c, q1, q2: dl * TDL + c * TC + q1 * TQ1 + a3 * TA3 + q2)(*d1(t))
           for dl in range(3) for a3 in range(N)]
    if b2_q1fast:
        d2 = lambda t: (t // 12, t % 4, (t // 4) % 3)                         # c, q1, a3
    else:
        d2 = lambda t: (t // 12, (t // 3) % 4, t % 3)
    b2l = [lambda t, dl=dl, q2=q2: (lambda c, q1, a3: dl * TDL + c * TC + q1 * TQ1 + a3 * TA3 + q2)(*d2(t))
           for dl in range(3) for q2 in (0, 2)]
    b2s = [lambda t, w=w, a2=a2: (lambda c, q1, a3: w * WW + c * WC + (a2 * 3 + a3) * WA + q1)(*d2(t))
           for w in range(2) for a2 in range(N)]
    b3l = [lambda t, w=w, q1=q1: w * WW + (t // 9) * WC + (t % 9) * WA + q1 for w in range(2) for q1 in (0, 2)]
    return dict(b1_st=cost(48, b1s), b2_ld=cost(36, b2l, 16), b2_st=cost(36, b2s), b3_ld=cost(27, b3l, 16))


def q3_stage2(perm):
    """3D Q3 (N = 4, Q = 6, 224-thread CTAs) stage-2 loads (LDS.128) and stores, per element;
    strides S1Q1 16, S1 96, fc 192 (stage 1), S2Q1 30, S2 180, fc 540 (stage 2)."""
    global NT
    nt, NT = NT, 224
    try:
        def dec(t):
            if not perm:
                return t // 24, (t // 4) % 6, t % 4
            pc, a3 = t >> 2, t & 3
            if pc < 24:
                return pc & 3, pc >> 2, a3
            r = pc - 24
            g, wi = r >> 2, r & 3
            return 4 + (wi & 1), g + (wi >> 1) * (4 if g < 2 else 1), a3
        ld = [lambda t, bg=bg, k=k: (lambda fc, q1, a3: fc * 192 + bg * 96 + q1 * 16 + a3 * 4 + 2 * k)(*dec(t))
              for bg in range(2) for k in range(2)]
        st = [lambda t, k=k, q2=q2: (lambda fc, q1, a3: fc * 540 + k * 180 + q1 * 30 + q2 * 4 + a3)(*dec(t))
              for k in range(3) for q2 in range(6)]
        return dict(stage2_ld=cost(144, ld, 16), stage2_st=cost(144, st))
    finally:
        NT = nt


def main():
    for perm in (False, True):
        print(f"Q3 stage 2, PERM_K3 = {int(perm)}: {q3_stage2(perm)}")
    for name, f, b in (("round-1 layout", (72, 36, 9, 144, 48, 12, "a3"), (144, 48, 12, 4, 108, 36, 4)),
                       ("LAYOUT_K2 = 1", (73, 36, 9, 147, 48, 12, "q1"), (150, 50, 12, 4, 162, 54, 6)),
                       ("+ XS_UNDER_K2", (105, 48, 12, 147, 48, 12, "q1"), (246, 82, 20, 6, 162, 54, 6, True))):
        fw, bw = forward(*f), backward(*b)
        print(f"{name:16s} forward {fw} backward {bw} total {sum(fw.values()) + sum(bw.values())}")


if __name__ == "__main__":
    main()
