"""The dispatch's division-by-reciprocal (csrc/fastdiv.h udiv_fast, used for the replica
index rho of reading A8) equals integer division on the whole range it is used for:
0 <= n < 2^31, 1 <= d < 2^31.  Compiled from the library header with g++ (host path)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SRC = r'''
#include <cstdio>
#include <cstdint>
#include <random>
#include "fastdiv.h"
int main() {
  std::mt19937_64 g(7);
  uint64_t bad = 0, n_checked = 0;
  auto chk = [&](uint32_t n, uint32_t d) {
    ++n_checked;
    if (moe::udiv_fast(n, d, 0xffffffffu / d) != n / d) ++bad;
  };
  for (uint32_t d = 1; d < 5000; ++d) {
    for (uint32_t n = 0; n < 3 * d + 3; ++n) chk(n, d);
    for (uint32_t n = 2147483647u; n > 2147483647u - 64; --n) chk(n, d);
    for (uint32_t q = 1; q < 64; ++q) { chk(q * d - 1, d); chk(q * d, d); chk(q * d + 1, d); }
  }
  for (int i = 0; i < 20000000; ++i) {
    const uint32_t d = 1 + (uint32_t)(g() % 2147483647u), n = (uint32_t)(g() % 2147483648u);
    chk(n, d);
    chk(n % (d + 1), d);
  }
  std::printf("%llu %llu\n", (unsigned long long)bad, (unsigned long long)n_checked);
  return bad != 0;
}
'''


def test_udiv_fast_equals_integer_division(tmp_path):
    src = tmp_path / "udiv.cpp"
    src.write_text(SRC)
    exe = tmp_path / "udiv"
    inc = ["-I", os.path.join(ROOT, "paper_2504_19925_b200", "csrc"), "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include"]
    r = subprocess.run(["g++", "-O2", "-std=c++17", *inc, str(src), "-o", str(exe)], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.fail(r.stderr[-2000:])
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    bad, n = (int(x) for x in out.stdout.split())
    assert bad == 0 and n > 40_000_000
