"""Mutation check of the oracle's pins: apply one plausible mistake at a time to
a throw-away copy of oracle/ and show that the CPU pins catch it.

    python tests/tools/mutate_oracle.py            # all mutations, prints one line each
    python tests/tools/mutate_oracle.py --list

Each mutation copies oracle/, tests/ and workloads/ to a temp dir, edits one line of
oracle/fbs_oracle.py, runs `pytest -m "not gpu"` on the oracle test files there and records
which tests fail.  A mutation that no test catches is reported as SURVIVED (exit code 1).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

# (name, old text, new text) — each old text must occur exactly once in oracle/fbs_oracle.py
MUTATIONS = [
    ("hier_init: multiply by P(1) instead of dividing",
     "w = [z_weight(k, alpha, beta) / P1[k] for k in range(pyr.K)]",
     "w = [z_weight(k, alpha, beta) * P1[k] for k in range(pyr.K)]"),
    # (z_weight(k + 1) at β = 0 scales every level by 1/α, which cancels in the quotient — the same
    # y_hier, so not a mistake; the shift that changes the result is the one below)
    ("hier_init: level index shifted in z_w (level k weighted as level k-1)",
     "w = [z_weight(k, alpha, beta) / P1[k] for k in range(pyr.K)]",
     "w = [z_weight(max(k - 1, 0), alpha, beta) / P1[k] for k in range(pyr.K)]"),
    ("hier_init: drop the top level",
     "den = P_project(pyr, [w[k] * PSc[k] for k in range(pyr.K)])",
     "den = P_project(pyr, [w[k] * PSc[k] * (k < pyr.K - 1) for k in range(pyr.K)])"),
    ("diagA: wrong B̄ diagonal (2 instead of 2D)",
     "diagA = lam * (m - n * bdiag * n) + Sc",
     "diagA = lam * (m - n * 2.0 * n) + Sc"),
    ("diagA: Sc dropped",
     "diagA = lam * (m - n * bdiag * n) + Sc",
     "diagA = lam * (m - n * bdiag * n)"),
    ("diagA: sign of the smoothness diagonal",
     "diagA = lam * (m - n * bdiag * n) + Sc",
     "diagA = lam * (n * bdiag * n - m) + Sc"),
    ("BT.601: R<->B swapped in U (BGR input)",
     "Un = -43 * r - 85 * g + 128 * b + 32768",
     "Un = -43 * b - 85 * g + 128 * r + 32768"),
    ("BT.601: R<->B swapped in V",
     "Vn = 128 * r - 107 * g - 21 * b + 32768",
     "Vn = 128 * b - 107 * g - 21 * r + 32768"),
    ("BT.601: U and V coefficient rows exchanged",
     "Un = -43 * r - 85 * g + 128 * b + 32768",
     "Un = 128 * r - 107 * g - 21 * b + 32768"),
    ("DT: schedule order reversed (narrowest kernel first)",
     "sigma_s * np.sqrt(3.0) * 2.0 ** (N - i) / np.sqrt(4.0 ** N - 1.0)",
     "sigma_s * np.sqrt(3.0) * 2.0 ** (i - 1) / np.sqrt(4.0 ** N - 1.0)"),
    ("DT: normalisation without the square root",
     "sigma_s * np.sqrt(3.0) * 2.0 ** (N - i) / np.sqrt(4.0 ** N - 1.0)",
     "sigma_s * np.sqrt(3.0) * 2.0 ** (N - i) / (4.0 ** N - 1.0)"),
    ("DT: base 4 instead of 2",
     "sigma_s * np.sqrt(3.0) * 2.0 ** (N - i) / np.sqrt(4.0 ** N - 1.0)",
     "sigma_s * np.sqrt(3.0) * 4.0 ** (N - i) / np.sqrt(4.0 ** N - 1.0)"),
]

TEST_FILES = ["tests/test_oracle.py", "tests/test_oracle_dt.py", "tests/test_oracle_d3.py",
              "tests/test_oracle_robust.py", "tests/test_oracle_lowrank.py"]


def run_one(name, old, new):
    src = open(os.path.join(ROOT, "oracle", "fbs_oracle.py")).read()
    assert src.count(old) == 1, f"mutation anchor not unique: {name}"
    with tempfile.TemporaryDirectory() as tmp:
        for d in ("oracle", "tests", "workloads"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("__pycache__"))
        with open(os.path.join(tmp, "oracle", "fbs_oracle.py"), "w") as fh:
            fh.write(src.replace(old, new))
        res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                              "-x" if "--fast" in sys.argv else "-q", *TEST_FILES],
                             cwd=tmp, capture_output=True, text=True)
        failed = [ln.split(" ")[1].split("::")[-1] for ln in res.stdout.splitlines() if ln.startswith("FAILED")]
        return res.returncode, failed


def main():
    if "--list" in sys.argv:
        for name, _, _ in MUTATIONS:
            print(name)
        return 0
    survived = 0
    for name, old, new in MUTATIONS:
        rc, failed = run_one(name, old, new)
        status = "caught" if rc != 0 else "SURVIVED"
        survived += rc == 0
        print(f"{status:8s} | {name} | failing: {', '.join(sorted(set(f.split('[')[0] for f in failed)))}")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
