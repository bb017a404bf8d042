"""Mutation check of the CPU oracle's pins ("chosen so that a plausible mistake
anywhere in it fails one of them").

Each mutation is one plausible slip in oracle/gvx_oracle_body.inc or gvx_oracle.c (a dropped
term, a wrong sign or index, a swapped operand, a wrong scale). For each one the repo's
tracked files are copied to a scratch directory, the mutation is applied there, and the
`-m "not gpu"` oracle tests run against the mutant (tests/conftest.py puts the scratch copy
first on sys.path, so `import oracle` builds and loads the mutated liboracle.so). Every
mutant must turn the suite red; the report says which test killed it.

    python tools/oracle_mutations.py [-j 8] [--out profiles/r02/oracle_mutations.txt]

Exit status 1 if any mutant survives. The unmutated copy is run first and must pass.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import re
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BODY = "oracle/gvx_oracle_body.inc"
MAIN = "oracle/gvx_oracle.c"
TESTS = ["tests/test_oracle_pins.py"]

# (name, file, old text, new text): `old` must occur exactly once.
MUTATIONS = [
    ("S x10 (boost tolerance scale)", BODY, "return g * (fabs(v[3]) + sqrt(b2) * p);",
     "return 10 * g * (fabs(v[3]) + sqrt(b2) * p);"),
    ("S without |beta| (gamma(E + |p|))", BODY, "return g * (fabs(v[3]) + sqrt(b2) * p);",
     "return g * (fabs(v[3]) + p);"),
    ("S without gamma", BODY, "return g * (fabs(v[3]) + sqrt(b2) * p);",
     "return (fabs(v[3]) + sqrt(b2) * p);"),
    ("S with beta^2 instead of |beta|", BODY, "return g * (fabs(v[3]) + sqrt(b2) * p);",
     "return g * (fabs(v[3]) + b2 * p);"),
    ("PtEtaPhiM E^2 clamp as sqrt|E^2|", BODY,
     "    T E2 = m * fabs(m) + pt * pt + pz * pz;\n    T E = sqrt(E2 > 0 ? E2 : (T)0);",
     "    T E2 = m * fabs(m) + pt * pt + pz * pz;\n    T E = sqrt(fabs(E2));"),
    ("PtEtaPhiM: no E^2 clamp (NaN)", BODY,
     "    T E2 = m * fabs(m) + pt * pt + pz * pz;\n    T E = sqrt(E2 > 0 ? E2 : (T)0);",
     "    T E2 = m * fabs(m) + pt * pt + pz * pz;\n    T E = sqrt(E2);"),
    ("PxPyPzM E^2 clamp as sqrt|E^2|", BODY,
     "    T E2 = px * px + py * py + pz * pz + m * fabs(m);\n    out[0] = px;\n    out[1] = py;\n"
     "    out[2] = pz;\n    out[3] = sqrt(E2 > 0 ? E2 : (T)0);",
     "    T E2 = px * px + py * py + pz * pz + m * fabs(m);\n    out[0] = px;\n    out[1] = py;\n"
     "    out[2] = pz;\n    out[3] = sqrt(fabs(E2));"),
    ("sin <-> cos in px, py", BODY, "    T px = pt * cos(phi);\n    T py = pt * sin(phi);",
     "    T px = pt * sin(phi);\n    T py = pt * cos(phi);"),
    ("pz with cosh instead of sinh", BODY, "    T pz = pt * sinh(eta);\n    T E2",
     "    T pz = pt * cosh(eta);\n    T E2"),
    ("drop m|m| from E^2", BODY, "T E2 = m * fabs(m) + pt * pt + pz * pz;", "T E2 = pt * pt + pz * pz;"),
    ("m*m instead of m|m|", BODY, "T E2 = m * fabs(m) + pt * pt + pz * pz;", "T E2 = m * m + pt * pt + pz * pz;"),
    ("drop pt^2 from E^2", BODY, "T E2 = m * fabs(m) + pt * pt + pz * pz;", "T E2 = m * fabs(m) + pz * pz;"),
    ("PtEtaPhiE: py from cos", BODY, "    out[1] = pt * sin(phi);\n    out[2] = pt * sinh(eta);\n    out[3] = E;",
     "    out[1] = pt * cos(phi);\n    out[2] = pt * sinh(eta);\n    out[3] = E;"),
    ("drop the spacelike sign", BODY, "return M2 >= 0 ? sqrt(M2) : -sqrt(-M2);", "return sqrt(fabs(M2));"),
    ("mass: drop pz^2 from |p|^2", BODY, "(w[0] * w[0] + w[1] * w[1] + w[2] * w[2])",
     "(w[0] * w[0] + w[1] * w[1])"),
    ("mass of the difference", BODY, "            w[k] = a[k] + b[k];\n        m_out[i] = FN(signed_mass_)(w);",
     "            w[k] = a[k] - b[k];\n        m_out[i] = FN(signed_mass_)(w);"),
    ("E_lab = E1 only", BODY, "            elab_out[i] = w[3];", "            elab_out[i] = a[3];"),
    ("Lambda: flip the sign of gamma*beta", BODY, "        L[i][3] = g * b[i];\n        L[3][i] = g * b[i];",
     "        L[i][3] = -g * b[i];\n        L[3][i] = -g * b[i];"),
    ("Lambda: g/(1+g) instead of g^2/(1+g)", BODY, "T bg = g * g / (1 + g);", "T bg = g / (1 + g);"),
    ("Lambda: (g-1) instead of g^2/(1+g)", BODY, "T bg = g * g / (1 + g);", "T bg = (g - 1);"),
    ("Lambda: swap beta_x, beta_y", BODY, "T b[3] = {bx, by, bz};", "T b[3] = {by, bx, bz};"),
    ("Lambda: b2 < 1 accepts |beta| = 1", BODY, "    *ok = (b2 < 1);", "    *ok = (b2 <= 1);"),
    ("apply: drop the time column", BODY, "        for (int j = 1; j < 4; ++j)\n            s = s + L[r][j] * v[j];",
     "        for (int j = 1; j < 3; ++j)\n            s = s + L[r][j] * v[j];"),
    ("CM: beta_cm = +P/E", BODY, "T bx = -P[0] / E, by = -P[1] / E, bz = -P[2] / E;",
     "T bx = P[0] / E, by = P[1] / E, bz = P[2] / E;"),
    ("CM: no E > 0 test", BODY, "    if (!(E > 0))\n        return NANT;\n    T bx", "    T bx"),
    ("CM: boosted vector 2 from vector 1", BODY, "    FN(apply_matrix_)(L, b, b2);", "    FN(apply_matrix_)(L, a, b2);"),
    ("histogram: CM flag ignored", BODY, "        if (cm) {\n            T bo[8];", "        if (0) {\n            T bo[8];"),
    ("cos theta*: p_y over |p|", BODY, "    T c = bo[2] / p;", "    T c = bo[1] / p;"),
    ("cos theta*: vector 2", BODY,
     "        T p = sqrt(bo[0] * bo[0] + bo[1] * bo[1] + bo[2] * bo[2]);\n        T c = bo[2] / p;",
     "        T p = sqrt(bo[4] * bo[4] + bo[5] * bo[5] + bo[6] * bo[6]);\n        T c = bo[6] / p;"),
    ("Lorentz: L transposed", BODY, "            L[r][c] = (T)Lrm[4 * r + c];", "            L[r][c] = (T)Lrm[4 * c + r];"),
    ("Lorentz: no metric check", BODY, "            if (fabs(m - want) > 1e-9 * (lmax * lmax > 1 ? lmax * lmax : 1))\n"
     "                return GVX_REF_DOMAIN;", "            (void)want;"),
    ("dimuon: same-sign pairs", BODY, "(int64_t)charge[first + 1] < 0)", "(int64_t)charge[first + 1] > 0)"),
    ("dimuon: >= 2 muons", BODY, "if (count == 2 &&", "if (count >= 2 &&"),
    ("dimuon: second muon = first", BODY,
     "            FN(load_cartesian_)(muons, 4, 1, first + 1, GVX_REF_PTETAPHIM, b);",
     "            FN(load_cartesian_)(muons, 4, 1, first, GVX_REF_PTETAPHIM, b);"),
    ("find_bin: no +1", MAIN, "    return 1 + (int32_t)(((double)nbins * (x - lo)) / (hi - lo));",
     "    return (int32_t)(((double)nbins * (x - lo)) / (hi - lo));"),
    ("find_bin: x <= lo is underflow", MAIN, "    if (x < lo)\n        return 0;", "    if (x <= lo)\n        return 0;"),
    ("find_bin: round instead of truncate", MAIN,
     "    return 1 + (int32_t)(((double)nbins * (x - lo)) / (hi - lo));",
     "    return 1 + (int32_t)round(((double)nbins * (x - lo)) / (hi - lo));"),
    ("find_bin: NaN to underflow", MAIN, "    if (x < lo)\n        return 0;", "    if (x < lo || x != x)\n        return 0;"),
    ("find_bin: hi edge inclusive", MAIN, "    if (!(x < hi))\n        return nbins + 1;",
     "    if (x > hi || x != x)\n        return nbins + 1;\n    if (x == hi)\n        return nbins;"),
]


def _tracked_files():
    out = subprocess.run(["git", "ls-files"], cwd=ROOT, check=True, capture_output=True, text=True).stdout
    return [f for f in out.splitlines() if f.split("/")[0] in ("oracle", "tests", "synth", "paper_2312_02756_b200")
            or f in ("pytest.ini", "setup.cfg", "pyproject.toml")]


def _copy_tree(dst: str):
    for f in _tracked_files():
        d = os.path.join(dst, f)
        os.makedirs(os.path.dirname(d), exist_ok=True)
        shutil.copy2(os.path.join(ROOT, f), d)


def _run(mut):
    name, path, old, new = mut if mut else ("(unmutated)", None, None, None)
    with tempfile.TemporaryDirectory(prefix="gvx_mut_") as tmp:
        _copy_tree(tmp)
        if path:
            p = os.path.join(tmp, path)
            src = open(p).read()
            if src.count(old) != 1:
                return name, "BAD-MUTATION", f"pattern occurs {src.count(old)} times"
            open(p, "w").write(src.replace(old, new))
        env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", "-m", "not gpu"]
                           + TESTS, cwd=tmp, env=env, capture_output=True, text=True, timeout=1800)
        failed = re.findall(r"^FAILED (\S+)", r.stdout, re.M)
        err = re.findall(r"^ERROR (\S+)", r.stdout, re.M)
        if r.returncode == 0:
            return name, "SURVIVED", r.stdout.strip().splitlines()[-1]
        return name, "killed", (failed or err or [r.stdout.strip().splitlines()[-1]])[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=min(8, os.cpu_count() or 1))
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    base = _run(None)
    lines = [f"baseline (unmutated oracle): {'passes' if base[1] == 'SURVIVED' else 'FAILS: ' + base[2]}"]
    ok = base[1] == "SURVIVED"
    with cf.ThreadPoolExecutor(args.j) as ex:
        res = list(ex.map(_run, MUTATIONS))
    for name, status, where in res:
        lines.append(f"{status:12s} {name:45s} {where}")
        ok = ok and status == "killed"
    killed = sum(s == "killed" for _, s, _ in res)
    lines.append(f"{killed}/{len(res)} mutants killed by {' + '.join(TESTS)} (-m 'not gpu')")
    text = "\n".join(lines) + "\n"
    print(text, end="")
    if args.out:
        os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
        with open(args.out, "w") as f:
            f.write(text)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
