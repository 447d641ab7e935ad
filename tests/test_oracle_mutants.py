"""Mutation check of the oracle's pins: plausible one-line bugs are injected into a
copy of oracle/lowdiff_ref.cpp, the copy is compiled and loaded in place of the oracle, and the
pin suite that covers the mutated part (-m "not gpu", stopping at the first failure) must fail.  A
mutant that survives means a pin is missing."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "lowdiff_ref.cpp")
C, X, F, U = ("tests/test_oracle_compress.py", "tests/test_oracle_exchange_optim.py", "tests/test_oracle_files.py",
              "tests/test_oracle_union.py")
A = "tests/test_oracle_accumulate.py"

MUTANTS = [
    ("ties go to the higher index", "      return a < b;\n    });", "      return a > b;\n    });", C),
    ("error-feedback add dropped", "acc[i] = ef ? residual[off + i] + grad[off + i] : grad[off + i];",
     "acc[i] = grad[off + i];", C),
    ("residual not zeroed at the selection", "for (uint64_t e = 0; e < k; ++e) residual[off + sel[e]] = 0.0f;",
     "for (uint64_t e = 0; e < k; ++e) residual[off + sel[e]] = residual[off + sel[e]];", C),
    ("k rounded up instead of down", "uint64_t k = (n * (uint64_t)ppm) / 1000000ull;",
     "uint64_t k = (n * (uint64_t)ppm + 999999ull) / 1000000ull;", C),
    ("merge overwrites instead of adding", "S[idx[e]] = S[idx[e]] + bits_float(val[e]);",
     "S[idx[e]] = bits_float(val[e]);", X),
    ("bias corrections swapped", "const float mh = m[j] * r1;\n    const float vh = v[j] * r2;",
     "const float mh = m[j] * r2;\n    const float vh = v[j] * r1;", X),
    ("beta^t off by one step", "for (int64_t i = 0; i < t; ++i) { p1 *= beta1; p2 *= beta2; }",
     "for (int64_t i = 0; i <= t; ++i) { p1 *= beta1; p2 *= beta2; }", X),
    ("incomplete full checkpoint accepted", "if (it->second.size() == world) { F = it->first; break; }",
     "if (!it->second.empty()) { F = it->first; break; }", F),
    ("mean not divided by N", "dense_out[j] = mean ? S[j] / n : S[j];", "dense_out[j] = S[j];", X),
    ("union keeps only the first rank's support",
     "for (int r = 0; r < world; ++r)\n    for (uint64_t e = 0; e < K; ++e) member[gathered[(uint64_t)r * 2 * K + e]] = 1;",
     "for (int r = 0; r < 1; ++r)\n    for (uint64_t e = 0; e < K; ++e) member[gathered[(uint64_t)r * 2 * K + e]] = 1;", U),
    ("accumulation overwrites instead of adding", "A[j] = before + x;", "A[j] = x;", A),
    ("accumulated batch replayed with its first iteration's step", "where[r][fe.first] = {fe.second, off, (int64_t)n_iters};",
     "where[r][fe.first] = {fe.second, off, 1};", A),
    ("CRC polynomial wrong", "(crc >> 1) ^ 0x82F63B78u", "(crc >> 1) ^ 0xEDB88320u", F),
]


@pytest.mark.parametrize("name,old,new,pins", MUTANTS, ids=[m[0] for m in MUTANTS])
def test_mutant_is_caught(tmp_path, name, old, new, pins):
    src = open(SRC).read()
    assert src.count(old) >= 1, f"mutation site for '{name}' not found"
    (tmp_path / "lowdiff_ref.cpp").write_text(src.replace(old, new))
    so = tmp_path / "liblowdiff_ref.so"
    subprocess.run(["g++", "-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-shared", "-o",
                    str(so), str(tmp_path / "lowdiff_ref.cpp")], check=True)
    env = dict(os.environ, LOWDIFF_REF_LIB=str(so))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", "-p", "no:cacheprovider", pins],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode != 0, f"mutant '{name}' survived every oracle pin:\n{r.stdout[-2000:]}"
