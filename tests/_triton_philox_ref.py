"""Independent Philox4x32-10 reference for the oracle pin: Triton's own `tl.philox`
(triton/language/random.py), executed by the Triton *CPU interpreter* (TRITON_INTERPRET=1).
Test-only; nothing in the product path imports Triton.

Usage: python _triton_philox_ref.py  < JSON [[c0,c1,c2,c3,k0,k1], ...]  > JSON [[x0..x3], ...]
"""
import json
import os
import sys

os.environ["TRITON_INTERPRET"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402
import triton  # noqa: E402
import triton.language as tl  # noqa: E402


@triton.jit
def _k(out_ptr, c_ptr, seed_ptr, N: tl.constexpr):
    i = tl.program_id(0)
    c0 = tl.load(c_ptr + i * 4 + 0)
    c1 = tl.load(c_ptr + i * 4 + 1)
    c2 = tl.load(c_ptr + i * 4 + 2)
    c3 = tl.load(c_ptr + i * 4 + 3)
    seed = tl.load(seed_ptr + i)
    a, b, c, d = tl.philox(seed, c0, c1, c2, c3)
    tl.store(out_ptr + i * 4 + 0, a)
    tl.store(out_ptr + i * 4 + 1, b)
    tl.store(out_ptr + i * 4 + 2, c)
    tl.store(out_ptr + i * 4 + 3, d)


def main():
    cases = json.load(sys.stdin)
    n = len(cases)
    ctr = np.array([[c[0], c[1], c[2], c[3]] for c in cases], dtype=np.uint32).view(np.int32)
    seeds = np.array([(c[5] << 32) | c[4] for c in cases], dtype=np.uint64).view(np.int64)
    out = torch.zeros(n * 4, dtype=torch.int32)
    _k[(n,)](out, torch.from_numpy(ctr.reshape(-1).copy()), torch.from_numpy(seeds.copy()), N=1)
    res = out.numpy().view(np.uint32).reshape(n, 4).tolist()
    json.dump(res, sys.stdout)


if __name__ == "__main__":
    main()
