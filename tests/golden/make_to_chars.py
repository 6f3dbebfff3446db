"""Golden vectors for format_number's real branch (instance.hpp:462-470 -> std::to_chars):
random doubles over many magnitudes printed by libstdc++'s std::to_chars. Needs g++ (C++17)."""
import os
import subprocess
import tempfile

import numpy as np

SRC = r"""
#include <charconv>
#include <cstdio>
int main(){ double v; char buf[64]; while (std::fread(&v, 8, 1, stdin) == 1) {
  auto r = std::to_chars(buf, buf + 64, v); *r.ptr = 0; std::printf("%s\n", buf); } }
"""

if __name__ == "__main__":
    rng = np.random.default_rng(1)
    v = np.concatenate([rng.random(4000) * 10.0 ** rng.integers(-30, 30, 4000), -rng.standard_normal(1000),
                        np.round(rng.random(1000) * 1000, 3), 10.0 ** np.arange(-20, 25),
                        [0.142, 1e-4, -0.001, 2.5e-7, 0.0, -0.0, 1e300, 5e-324]])
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "t.cpp"), os.path.join(d, "t")
        open(src, "w").write(SRC)
        subprocess.run(["g++", "-std=c++17", "-O2", "-o", exe, src], check=True)
        out = subprocess.run([exe], input=v.astype(np.float64).tobytes(), capture_output=True, check=True)
    text = out.stdout.decode().split()
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "to_chars_vectors.npz"),
                        values=v, text=np.array(text))
