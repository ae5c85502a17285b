"""Pins of the oracle's Philox4x32-10 and of the mask drawn from it (reading R17), with no GPU:
the generator's published known-answer vectors, NVIDIA's independent host implementation
(curand_Philox4x32_10 from the CUDA toolkit headers, compiled here for the CPU), agreement of the
vectorised and the big-integer versions, and the mask layout (pairs of coefficients per draw,
uniform range, counter fields)."""
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import philox

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden" / "philox4x32_10_kat.txt"


def _kat():
    rows = []
    for line in GOLD.read_text().splitlines():
        if line.strip() and not line.startswith("#"):
            v = [int(x, 16) for x in line.split()]
            rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


def test_known_answer_vectors():
    rows = _kat()
    assert len(rows) == 3
    for ctr, key, out in rows:
        assert philox.philox4x32_10_int(ctr, key) == out
        got = [int(np.asarray(w).item()) for w in philox.philox4x32_10(ctr, key)]
        assert got == out


_CURAND = r"""
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
#include <cstdio>
#include <cstdlib>
int main(int argc, char** argv) {
  unsigned s = 12345u;
  for (int i = 0; i < 2000; ++i) {
    unsigned v[6];
    for (int k = 0; k < 6; ++k) { s = s * 1664525u + 1013904223u; v[k] = s ^ (s >> 13) * (i & 7); }
    if (i < 4) for (int k = 0; k < 6; ++k) v[k] = i == 0 ? 0u : i == 1 ? 0xffffffffu : (unsigned)(i * 0x10001 + k);
    uint4 c = make_uint4(v[0], v[1], v[2], v[3]);
    uint2 key = make_uint2(v[4], v[5]);
    uint4 o = curand_Philox4x32_10(c, key);
    printf("%08x %08x %08x %08x %08x %08x %08x %08x %08x %08x\n", v[0], v[1], v[2], v[3], v[4], v[5], o.x, o.y, o.z, o.w);
  }
  return 0;
}
"""


def test_matches_curand_host_implementation(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(nvcc).exists():
        pytest.skip("nvcc not available")
    src = tmp_path / "ph.cu"
    src.write_text(_CURAND)
    exe = tmp_path / "ph"
    subprocess.check_call([nvcc, "-O1", "-o", str(exe), str(src)], cwd=tmp_path)
    lines = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    rows = [[int(x, 16) for x in l.split()] for l in lines if l.strip()]
    assert len(rows) == 2000
    arr = np.array(rows, dtype=np.uint64)
    got = philox.philox4x32_10(tuple(arr[:, k] for k in range(4)), (arr[:, 4], arr[:, 5]))
    for k in range(4):
        assert (got[k] == arr[:, 6 + k]).all()
    for r in rows[:50]:
        assert philox.philox4x32_10_int(r[0:4], r[4:6]) == r[6:10]


def test_mask_layout_and_range():
    seed, stream, n, tb = 0x0123456789ABCDEF, 7, 64, 37
    r = philox.mask(seed, stream, 3, n, tb, ct0=5)
    assert r.shape == (3, n) and r.dtype == np.uint64 and int(r.max()) < (1 << tb)
    for i in range(3):
        for e in (0, 1, 2, 63):
            w = philox.philox4x32_10_int((e >> 1, 5 + i, stream, 0), (seed & 0xFFFFFFFF, seed >> 32))
            lo, hi = (w[0], w[1]) if e % 2 == 0 else (w[2], w[3])
            assert int(r[i, e]) == ((hi << 32) | lo) & ((1 << tb) - 1)
    # slices of the output index space agree with the whole (the rank-slice property)
    full = philox.mask(seed, stream, 8, n, tb)
    assert (philox.mask(seed, stream, 3, n, tb, ct0=5) == full[5:8]).all()
    # different streams / seeds give different masks
    assert (philox.mask(seed, stream + 1, 1, n, tb) != full[:1]).any()
    assert (philox.mask(seed + 1, stream, 1, n, tb) != full[:1]).any()


def test_mask_is_uniform_looking():
    """Coarse sanity of the draw: every one of the 37 bits is set about half the time."""
    r = philox.mask(99, 1, 4, 4096, 37)
    bits = np.array([((r >> np.uint64(b)) & np.uint64(1)).mean() for b in range(37)])
    assert np.all(np.abs(bits - 0.5) < 0.02)
