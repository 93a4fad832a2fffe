"""The exact star kernel divides by the Jacobi divisor D with a host-computed y = RN(1/D):
q0 = RN(a*y), r = fma(-D, q0, a), q = fma(r, y, q0) (star_exact.cuh xdiv).  Markstein's
theorem says q is the correctly rounded a/D when every intermediate is normal; this test
checks the identity against IEEE division (what numpy's `/` gives, executor.py:96) for the
divisors the corpus kernels use and for random ones, over the magnitude range the kernel
takes the fast path for (|a| in (2^-900, 2^900), |D| in [2^-64, 2^64]) — compiled C with a
correctly rounded fma(), no GPU."""

from __future__ import annotations

import shutil
import subprocess

import pytest

from paper_2309_04671_b200 import front

SRC = r"""
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
static uint64_t s = 0x9E3779B97F4A7C15ull;
static uint64_t nx(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static double rnd(int emin, int emax) {
    uint64_t m = nx() & ((1ull << 52) - 1);
    int e = emin + (int)(nx() % (uint64_t)(emax - emin + 1));
    uint64_t b = ((uint64_t)(e + 1023) << 52) | m;
    double d; memcpy(&d, &b, 8);
    return (nx() & 1) ? -d : d;
}
static long check(double D, long n) {
    double y = 1.0 / D; long bad = 0;
    for (long t = 0; t < n; ++t) {
        double a = rnd(-899, 899);
        double q0 = a * y, r = fma(-D, q0, a), q = fma(r, y, q0), ref = a / D;
        if (memcmp(&q, &ref, 8)) ++bad;
    }
    return bad;
}
int main(int argc, char** argv) {
    long n = atol(argv[1]), bad = 0;
    for (int i = 2; i < argc; ++i) bad += check(atof(argv[i]), n);
    for (int k = 0; k < 200; ++k) bad += check(fabs(rnd(-64, 63)), n / 10);
    printf("%ld\n", bad);
    return 0;
}
"""


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_reciprocal_division_is_correctly_rounded(tmp_path):
    sk_corpus = front.module("corpus")
    divisors = set()
    for k in sk_corpus.TABLE_KERNELS:  # the normalised corpus kernels divide by their coefficient sum
        text = sk_corpus.source_text(k.name)
        if ") / " in text:
            divisors.add(text.split(") / ")[1].split(")")[0].split()[0].rstrip(","))
    from paper_2309_04671_b200 import corpus

    for name in ("star3d1r_norm", "star3d2r_norm", "star3d3r_norm", "star3d4r_norm"):  # c2-c5's divisors
        divisors.add(corpus.kernel_source(name)[3].rsplit("/", 1)[1].strip())
    assert len(divisors) >= 8
    divisors |= {"3", "7", "0.1", "1.9999999999999998", "1.0000000000000002"}
    (tmp_path / "x.c").write_text(SRC)
    exe = tmp_path / "x"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", str(exe), str(tmp_path / "x.c"), "-lm"], check=True)
    out = subprocess.run([str(exe), "200000", *sorted(divisors)], capture_output=True, text=True, check=True)
    assert out.stdout.strip() == "0"
