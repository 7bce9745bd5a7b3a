"""Generate paper_2310_15419_b200/csrc/bm_tables.h -- constants of the fast fp64 Box-Muller
transform (philox.cuh: bm_m2log_u53 / bm_sincos) -- and check the method against 300-bit mpmath.

    python scripts/gen_bm_tables.py [--check N]

Product-side only: the oracle keeps libm's log / sqrt / cos / sin (oracle/sketch_oracle.c); the
GPU parity tests compare the two within 1e-14 relative (Gaussian row).

-2 log(u1), u1 = K 2^-53 with K = k1 + 1 in [1, 2^53] (bm_m2log_u53):  K = 2^e m, m in [1, 2);
  idx = round(128 (m - 1)) in [0, 128]; c = 1 / (1 + idx/128) rounded to 12 significant bits
  (c_0 = 1, c_128 = 1/2 exactly); table rows {-2c, 2 L_hi, 2 L_lo} with L = log c split so L_hi and
  ln2_hi are multiples of 2^-42 (the first bracket below is exact);  s = fma(m, -2c, 2) = -2 (m c - 1)
  exactly (|s| < 0.009), -2 log u1 = (e (-2 ln2_hi) + 2 L_hi) + (s + s^2 Q(s) + (e (-2 ln2_lo) + 2 L_lo)),
  Q(s) = 1/4 + s/12 + s^2/32 + s^3/80 + s^4/192 (= -P(-s/2)/2 for the Taylor P of (log1p(r) - r) / r^2;
  the s^5/448 term is below 2^-60 relative), so Box-Muller's factor -2 costs no multiply.
sin / cos by table (bm_sincos): j = rint(256 theta / pi) in [0, 512], r = theta - j pi/256 (pi/256
  in three parts, j pi/256 exact for the first two), |r| <= pi/512; sin r = r + r^3 (-1/6 + r^2/120),
  cos r = 1 + r^2 (-1/2 + r^2/24) (Taylor; the next terms are below 2^-55 relative on this interval);
  sin theta = S_j cos r + C_j sin r, cos theta = C_j cos r - S_j sin r with S_j, C_j = sin, cos (j pi/256)
  correctly rounded (exact zeros at multiples of pi/2, so no cancellation near the zeros of sin and cos).
"""
import argparse
import os
import random
import struct

import mpmath as mp
import numpy as np

mp.mp.prec = 300
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "paper_2310_15419_b200", "csrc", "bm_tables.h")

def hexd(x: float) -> str:
    return "0x%016xull" % struct.unpack("<Q", struct.pack("<d", x))[0]


def round_bits(x, bits):
    """Round mpf x to a double with at most `bits` significant bits."""
    e = int(mp.floor(mp.log(abs(x), 2)))
    q = mp.mpf(2) ** (e - bits + 1)
    return float(mp.nint(x / q) * q)


def round_grid(x, g):
    return float(mp.nint(x * mp.mpf(2) ** g) / mp.mpf(2) ** g)


LN2 = mp.log(2)
LN2_HI = round_grid(LN2, 42)
LN2_LO = float(LN2 - LN2_HI)
NSC = 512                                      # sin / cos table intervals over [0, 2 pi)
PISC = 2 * mp.pi / NSC
PISC_0 = round_bits(PISC, 43)                  # j * PISC_0 exact for j <= 512 (10 + 43 bits)
PISC_1 = round_bits(PISC - PISC_0, 43)
PISC_2 = float(PISC - PISC_0 - PISC_1)
SC_TAB = [(float(mp.sin(j * PISC)), float(mp.cos(j * PISC))) for j in range(NSC + 1)]
for j in range(0, NSC + 1, NSC // 4):          # exact zeros / ones at multiples of pi/2
    SC_TAB[j] = (float(mp.nint(mp.sin(j * PISC))), float(mp.nint(mp.cos(j * PISC))))


def fma(a, b, c):
    return float(mp.mpf(a) * mp.mpf(b) + mp.mpf(c))


def bm_sincos_tab(th: float):
    """float64 emulation (with fma) of philox.cuh bm_sincos."""
    kr = fma(th, float(1 / PISC), 6755399441055744.0)
    kd = kr - 6755399441055744.0
    j = int(kd)
    r = fma(-kd, PISC_0, th)
    r = fma(-kd, PISC_1, r)
    r = fma(-kd, PISC_2, r)
    S, C = SC_TAB[j]
    z = r * r
    ps = fma(z, 1.0 / 120.0, -1.0 / 6.0)
    sr = fma(z * r, ps, r)
    cr = fma(z, fma(z, 1.0 / 24.0, -0.5), 1.0)
    return fma(S, cr, C * sr), fma(C, cr, -(S * sr))


def table():
    rows = []
    for i in range(129):
        c = round_bits(1 / (1 + mp.mpf(i) / 128), 12)
        if i == 128:
            hi, lo = -LN2_HI, -LN2_LO
        else:
            L = mp.log(mp.mpf(c))
            hi = round_grid(L, 42)
            lo = float(L - hi)
        rows.append((c, hi, lo))
    assert rows[0] == (1.0, 0.0, 0.0) and rows[128][0] == 0.5
    return rows


Q = [1 / 4, 1 / 12, 1 / 32, 1 / 80, 1 / 192, 1 / 448]


def bm_m2log_u53(K: int, rows) -> float:
    """float64 emulation (with fma) of philox.cuh bm_m2log_u53: -2 log(K 2^-53), 1 <= K <= 2^53."""
    U = float(K)
    b = struct.unpack("<Q", struct.pack("<d", U))[0]
    e = ((b >> 52) & 0x7FF) - 1023 - 53
    m = struct.unpack("<d", struct.pack("<Q", (b & ((1 << 52) - 1)) | (0x3FF << 52)))[0]
    idx = (((b >> 44) & 0xFF) + 1) >> 1
    c, hi, lo = rows[idx]
    sv = fma(m, -2.0 * c, 2.0)
    q = fma(sv, Q[4], Q[3])                      # degree 4: the s^5 / 448 term is below 2^-60 relative
    for k in (2, 1, 0):
        q = fma(sv, q, Q[k])
    shi = fma(float(e), -2.0 * LN2_HI, 2.0 * hi)
    slo = fma(float(e), -2.0 * LN2_LO, 2.0 * lo)
    return shi + (sv + fma(sv * sv, q, slo))


def check(n: int, rows) -> None:
    rng = random.Random(5)
    worst_m2 = 0.0
    Ks = [rng.randrange(1, 2 ** 53 + 1) for _ in range(n)] + [1, 2, 2 ** 52, 2 ** 53, 2 ** 53 - 1]
    Ks += [2 ** 53 - k for k in range(1, 200)] + [2 ** 52 + k for k in range(-50, 50)]
    for ex in range(45, 53):                     # mantissas at the table's rounding boundaries
        for i in range(128):
            Ks += [int((1 + (2 * i + 1) / 256) * 2 ** ex) + dk for dk in (-1, 0, 1)]
    for K in Ks:
        ref = -2 * mp.log(mp.mpf(K) * mp.mpf(2) ** -53)
        got = bm_m2log_u53(K, rows)
        if ref != 0:
            worst_m2 = max(worst_m2, float(abs((got - ref) / ref)))
        else:
            assert got == 0.0
    print(f"-2 log(u1) max rel error {worst_m2:.3g}")
    assert worst_m2 < 8 * 2.0 ** -53
    # table sincos over theta = u2 fl(2 pi), u2 = k 2^-53 (random k, and k near the multiples of
    # 2^51 = the quadrant boundaries where sin or cos vanishes)
    two_pi = 6.283185307179586
    ks = [rng.randrange(0, 2 ** 53) for _ in range(n)]
    ks += [q * 2 ** 51 + dk for q in range(4) for dk in range(-40, 41) if 0 <= q * 2 ** 51 + dk < 2 ** 53]
    ks += [2 ** 53 - 1, 1, 2, 3]
    worst_ts = worst_tc = 0.0
    for k in ks:
        th = (k * 2.0 ** -53) * two_pi                              # u2 fl(2 pi), one IEEE multiply
        s, c = bm_sincos_tab(th)
        rs, rc = mp.sin(mp.mpf(th)), mp.cos(mp.mpf(th))
        if rs != 0:
            worst_ts = max(worst_ts, float(abs((s - rs) / rs)))
        if rc != 0:
            worst_tc = max(worst_tc, float(abs((c - rc) / rc)))
    print(f"table sincos max rel error: sin {worst_ts:.3g}, cos {worst_tc:.3g}")
    assert worst_ts < 16 * 2.0 ** -53 and worst_tc < 16 * 2.0 ** -53


def write(rows) -> None:
    lines = ["// bm_tables.h -- GENERATED by scripts/gen_bm_tables.py; do not edit.",
             "// Constants of the fast fp64 Box-Muller transform (philox.cuh): the -2 log table (c_i, log c_i",
             "// as hi + lo with hi on the 2^-42 grid), ln 2 split the same way, pi/256 in three parts and the",
             "// sin / cos table.  Product code only (the oracle uses libm).",
             "#pragma once", "#include <cstdint>", "", "namespace sk {", "",
             "// Scalar constants live in the constant bank so DFMA / DMUL read them as c[][] operands",
             "// (fp64 immediates would be rebuilt with UMOV pairs at every use).",
             "enum BmK { kRound, kSCInv, kSCPi_0, kSCPi_1, kSCPi_2, kT3, kT5, kU2, kU4,",
             "           kQ0, kQ1, kQ2, kQ3, kQ4, kM2Ln2Hi, kM2Ln2Lo, kTwoPi53, kBmKCount };",
             "__device__ __constant__ double kBm[kBmKCount] = {",
             "    6755399441055744.0 /* 1.5 2^52: rint by addition */,",
             f"    {float(1 / PISC)!r}, {PISC_0!r}, {PISC_1!r}, {PISC_2!r},",
             "    -1.0 / 6.0, 1.0 / 120.0, -0.5, 1.0 / 24.0,",
             "    1.0 / 4.0, 1.0 / 12.0, 1.0 / 32.0, 1.0 / 80.0, 1.0 / 192.0,",
             f"    {-2.0 * LN2_HI!r}, {-2.0 * LN2_LO!r}, {6.283185307179586 * 2.0 ** -53!r} /* fl(2 pi) 2^-53 */}};",
             "", "// {-2 c_i, 2 log(c_i)_hi, 2 log(c_i)_lo}, i = 0..128: the table of log u scaled for -2 log u",
             "// (bm_m2log_u53; the kernels copy it to shared memory)",
             "constexpr int kBmLogRows = 129;",
             "__device__ const double kBmLogTab[kBmLogRows][3] = {"]
    for c, hi, lo in rows:
        lines.append(f"    {{{-2.0 * c!r}, {2.0 * hi!r}, {2.0 * lo!r}}},")
    lines += ["};", "", f"// {{sin(j 2pi/{NSC}), cos(j 2pi/{NSC})}}, j = 0..{NSC}, correctly rounded (exact 0 / +-1 at multiples of pi/2)",
              f"constexpr int kBmSinCosN = {NSC};",
              f"__device__ const double kBmSinCosTab[{NSC + 1}][2] = {{"]
    for sv, cv in SC_TAB:
        lines.append(f"    {{{sv!r}, {cv!r}}},")
    lines += ["};", "", "}  // namespace sk", ""]
    with open(OUT, "w") as f:
        f.write("\n".join(lines))
    print("wrote", OUT)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--check", type=int, default=20000)
    a = ap.parse_args()
    rows = table()
    check(a.check, rows)
    write(rows)
