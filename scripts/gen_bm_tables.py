"""Generate paper_2310_15419_b200/csrc/bm_tables.h -- constants of the fast fp64 Box-Muller
transform (philox.cuh: bm_log / bm_sincos) -- and check the method against 300-bit mpmath.

    python scripts/gen_bm_tables.py [--check N]

Product-side only: the oracle keeps libm's log / sqrt / cos / sin (oracle/sketch_oracle.c); the
GPU parity tests compare the two within 1e-14 relative (Gaussian row).

log(u), u in (0, 1]:  u = 2^e m, m in [1, 2); idx = round(128 (m - 1)) in [0, 128];
  c = 1 / (1 + idx/128) rounded to 12 significant bits (c_0 = 1, c_128 = 1/2 exactly);
  r = fma(m, c, -1), |r| < 0.0045;  log u = (e ln2_hi - L_hi) + (r + r^2 P(r) + (e ln2_lo - L_lo))
  with L = log(c) split so that L_hi and ln2_hi are multiples of 2^-42 (the first bracket is exact)
  and P the Taylor polynomial of (log1p(r) - r) / r^2 to degree 5.
sin / cos on |r| <= pi/4 after the Cody-Waite reduction r = theta - k pi/2 (pi/2 in four parts):
  the minimax kernels of fdlibm (Sun Microsystems, 1993; public domain), error < 1 ulp.
-2 log(u1) directly (bm_m2log_u53, the form in use): the same table scaled by -2 / 2 (rows {-2c,
  2 L_hi, 2 L_lo}), s = fma(m, -2c, 2) = -2r exactly, and Q(s) = -P(-s/2)/2 = 1/4 + s/12 + s^2/32
  + s^3/80 + s^4/192 (+ s^5/448, dropped: same worst case 1.3e-16 over random and idx-boundary
  inputs), so the factor -2 of Box-Muller costs no multiply; u1 enters as
  the integer k1 + 1 (exponent bias 53) and theta = k2 (2^-53 fl(2 pi)), one multiply each.
sin / cos by table (bm_sincos, the one in use): j = rint(256 theta / pi) in [0, 512],
  r = theta - j pi/256 (pi/256 in three parts, j pi/256 exact for the first two), |r| <= pi/512;
  sin r = r + r^3 (-1/6 + r^2/120), cos r = 1 + r^2 (-1/2 + r^2/24) (Taylor; the next terms are
  below 2^-55 relative on this interval); sin theta = S_j cos r + C_j sin r,
  cos theta = C_j cos r - S_j sin r with S_j, C_j = sin, cos (j pi/256) correctly rounded (exact
  zeros at multiples of pi/2, so no cancellation near the zeros of sin and cos).
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

S = [-1.66666666666666324348e-01, 8.33333333332248946124e-03, -1.98412698298579493134e-04,
     2.75573137070700676789e-06, -2.50507602534068634195e-08, 1.58969099521155010221e-10]
C = [4.16666666666666019037e-02, -1.38888888888741095749e-03, 2.48015872894767294178e-05,
     -2.75573143513906633035e-07, 2.08757232129817482790e-09, -1.13596475577881948265e-11]


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


def bm_log(u: float, rows) -> float:
    """float64 emulation (no fma: one extra rounding in r) of bm_log."""
    b = struct.unpack("<Q", struct.pack("<d", u))[0]
    e = ((b >> 52) & 0x7FF) - 1023
    m = struct.unpack("<d", struct.pack("<Q", (b & ((1 << 52) - 1)) | (0x3FF << 52)))[0]
    idx = (((b >> 44) & 0xFF) + 1) >> 1
    c, hi, lo = rows[idx]
    r = float(mp.mpf(m) * c - 1)                  # fma
    p = -1 / 2 + r * (1 / 3 + r * (-1 / 4 + r * (1 / 5 + r * (-1 / 6 + r * (1 / 7)))))
    return (e * LN2_HI - hi) + (r + (r * r * p + (e * LN2_LO - lo)))


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


def kernels(r: float):
    z = r * r
    v = z * r
    ps = S[1] + z * (S[2] + z * (S[3] + z * (S[4] + z * S[5])))
    s = r + v * (S[0] + z * ps)
    pc = z * (C[0] + z * (C[1] + z * (C[2] + z * (C[3] + z * (C[4] + z * C[5])))))
    hz = 0.5 * z
    w = 1.0 - hz
    c = w + (((1.0 - w) - hz) + z * pc)
    return s, c


def check(n: int, rows) -> None:
    rng = random.Random(5)
    worst_log = worst_s = worst_c = 0.0
    us = [rng.randrange(1, 2 ** 53 + 1) * 2.0 ** -53 for _ in range(n)]
    us += [1.0, 1 - 2.0 ** -53, 2.0 ** -53, 0.5, 0.5 - 2.0 ** -54, 1 - 2.0 ** -9, 1 - 2.0 ** -8]
    us += [1 - k * 2.0 ** -53 for k in range(1, 200)]
    for u in us:
        ref = mp.log(mp.mpf(u))
        got = bm_log(u, rows)
        if ref != 0:
            worst_log = max(worst_log, float(abs((got - ref) / ref)))
        else:
            assert got == 0.0
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
    for _ in range(n):
        r = rng.uniform(-float(mp.pi / 4), float(mp.pi / 4))
        s, c = kernels(r)
        worst_s = max(worst_s, float(abs((s - mp.sin(r)) / mp.sin(r))))
        worst_c = max(worst_c, float(abs((c - mp.cos(r)) / mp.cos(r))))
    print(f"max rel error: log {worst_log:.3g}, sin kernel {worst_s:.3g}, cos kernel {worst_c:.3g} "
          f"(2^-52 = {2.0 ** -52:.3g})")
    assert worst_log < 8 * 2.0 ** -53 and worst_s < 4 * 2.0 ** -53 and worst_c < 4 * 2.0 ** -53
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
             "// Constants of the fast fp64 Box-Muller transform (philox.cuh): log table (c_i, log c_i as",
             "// hi + lo with hi on the 2^-42 grid), ln 2 split the same way, pi/2 in four parts (Cody-Waite)",
             "// and the fdlibm sin / cos kernel coefficients.  Product code only (the oracle uses libm).",
             "#pragma once", "#include <cstdint>", "", "namespace sk {", "",
             "// Scalar constants live in the constant bank so DFMA / DMUL read them as c[][] operands",
             "// (fp64 immediates would be rebuilt with UMOV pairs at every use).",
             "enum BmK { kLn2Hi, kLn2Lo, kPio2_0, kPio2_1, kPio2_2, kPio2_3, kS1, kS2, kS3, kS4, kS5, kS6,",
             "           kC1, kC2, kC3, kC4, kC5, kC6, kL7, kL6, kL5, kL4, kL3, kL2, kTwoOverPi, kRound, kTwoPi,",
             "           kSCInv, kSCPi_0, kSCPi_1, kSCPi_2, kT3, kT5, kT7, kU2, kU4, kU6,",
             "           kQ0, kQ1, kQ2, kQ3, kQ4, kQ5, kM2Ln2Hi, kM2Ln2Lo, kTwoPi53, kBmKCount };",
             "__device__ __constant__ double kBm[kBmKCount] = {",
             f"    {LN2_HI!r}, {LN2_LO!r},",
             "    1.57079632673412561417e+00, 6.07710050630396597660e-11, 2.02226624871116645580e-21,",
             "    8.47842766036889956997e-32,",
             "    " + ", ".join(repr(x) for x in S) + ",",
             "    " + ", ".join(repr(x) for x in C) + ",",
             "    1.0 / 7.0, -1.0 / 6.0, 1.0 / 5.0, -1.0 / 4.0, 1.0 / 3.0, -0.5,",
             "    0.63661977236758138243, 6755399441055744.0, 6.283185307179586 /* fl(2 pi) */,",
             f"    {float(1 / PISC)!r}, {PISC_0!r}, {PISC_1!r}, {PISC_2!r},",
             "    -1.0 / 6.0, 1.0 / 120.0, -1.0 / 5040.0, -0.5, 1.0 / 24.0, -1.0 / 720.0,",
             "    1.0 / 4.0, 1.0 / 12.0, 1.0 / 32.0, 1.0 / 80.0, 1.0 / 192.0, 1.0 / 448.0,",
             f"    {-2.0 * LN2_HI!r}, {-2.0 * LN2_LO!r}, {6.283185307179586 * 2.0 ** -53!r} /* fl(2 pi) 2^-53 */}};",
             "", "// {-2 c_i, 2 log(c_i)_hi, 2 log(c_i)_lo, 0}, i = 0..128 (32-byte rows; copied to shared memory):",
             "// the table of log u scaled for -2 log u (bm_m2log_u53)",
             "__device__ const double kBmLogTab[129][4] = {"]
    for c, hi, lo in rows:
        lines.append(f"    {{{-2.0 * c!r}, {2.0 * hi!r}, {2.0 * lo!r}, 0.0}},")
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
