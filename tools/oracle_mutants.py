"""Mutation check of the oracle's pins (CPU only; not part of the product).

Applies one plausible mistake at a time to a COPY of oracle/abft_oracle.c (a
dropped term, a wrong sign or index, a transposed operand, an unrounded
operand, a missing repair ...), rebuilds that copy's liboracle.so and runs
the `-m "not gpu"` oracle pins against it.  A mutant that no pin fails is a
gap in the pins.  Usage (from the repo root):

    python tools/oracle_mutants.py [--out profiles/.../oracle_mutants.txt]
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, passage, old text, new text) -- each old text must occur exactly once
MUTANTS = [
    ("clamp reads the far edge", "P:289-292", "if (bc == OR_BC_CLAMP) return c < 0 ? 0 : n - 1;",
     "if (bc == OR_BC_CLAMP) return c < 0 ? n - 1 : 0;"),
    ("periodic wrap without +n", "P:407-412", "return ((c % n) + n) % n;", "return c % n;"),
    ("constant ghost read as 0", "P:413-415", "return p->bc == OR_BC_CONSTANT ? rnd(p->dtype, p->bc_value) : 0.0;",
     "return 0.0;"),
    ("cell index transposed", "Eq. 1", "return ld(u, (zr * p->ny + yr) * p->nx + xr, p->dtype);",
     "return ld(u, (zr * p->nx + xr) * p->ny + yr, p->dtype);"),
    ("flip of the next bit", "P:783-785", "b ^= (uint32_t)1u << bit;", "b ^= (uint32_t)1u << (bit + 1);"),
    ("fp32 chain unfused", "Q23", "acc = (k == 0) ? w * v : fmaf(w, v, acc);", "acc = (k == 0) ? w * v : acc + w * v;"),
    ("fp32 source term unfused", "Q23", "acc = fmaf(cf, sv, acc);", "acc = acc + cf * sv;"),
    ("fp64 weight sign", "Eq. 1", "acc = (k == 0) ? q->w * v : fma(q->w, v, acc);",
     "acc = (k == 0) ? q->w * v : fma(-q->w, v, acc);"),
    ("fp64 source dropped", "Eq. 1", "acc = fma(s->coef, sv, acc);", "acc = acc;"),
    ("flip one sweep late", "P:785", "if (!F->armed || F->sweep != sweep) continue;",
     "if (!F->armed || F->sweep != sweep - 1) continue;"),
    ("flip fires twice", "Q18", "faults[g].x == F->x && faults[g].armed == -1) dup = 1;",
     "faults[g].x == F->x && faults[g].armed == -2) dup = 1;"),
    ("a sums a row", "Eq. 2", "for (int64_t y = 0; y < ny; y++) s += ld(u, (z * ny + y) * nx + x, p->dtype);\n      A[z * nx + x] = s;",
     "for (int64_t y = 0; y < ny; y++) s += ld(u, (z * ny + x % ny) * nx + y % nx, p->dtype);\n      A[z * nx + x] = s;"),
    ("b skips the last column", "Eq. 3", "for (int64_t x = 0; x < nx; x++) s += ld(u, (z * ny + y) * nx + x, p->dtype);\n      B[z * ny + y] = s;",
     "for (int64_t x = 0; x < nx - 1; x++) s += ld(u, (z * ny + y) * nx + x, p->dtype);\n      B[z * ny + y] = s;"),
    ("c: terms subtracted", "P:321", "s = (k == 0) ? t : s + t;", "s = (k == 0) ? t : s - t;"),
    ("c: unrounded coefficient", "P:321, Q23", "double cf = rnd(p->dtype, q->coef);", "double cf = q->coef;"),
    ("c: unrounded scalar", "P:321, Q23", "double sv = q->field ? ld(q->field, c, p->dtype) : rnd(p->dtype, q->scalar);",
     "double sv = q->field ? ld(q->field, c, p->dtype) : q->scalar;"),
    ("c_y sums a column", "P:321", "for (int64_t x = 0; x < nx; x++) s += cval(p, (z * ny + y) * nx + x);",
     "for (int64_t x = 0; x < nx; x++) s += cval(p, (z * ny + (x % ny)) * nx + (y % nx));"),
    ("alpha: one ghost row short", "P:323-326", "for (int64_t y = j; y <= -1; y++) s1 += val(p, u, z, y, x);",
     "for (int64_t y = j + 1; y <= -1; y++) s1 += val(p, u, z, y, x);"),
    ("alpha: sign", "P:323-326", "  return s1 - s2;\n}\n\n/* beta", "  return s2 - s1;\n}\n\n/* beta"),
    ("alpha: j>0 one row long", "P:323-326", "for (int64_t y = ny; y <= ny + j - 1; y++) s1 += val(p, u, z, y, x);",
     "for (int64_t y = ny; y <= ny + j; y++) s1 += val(p, u, z, y, x);"),
    ("beta: sign", "P:327-332", "    for (int64_t x = 0; x <= i - 1; x++) s2 += val(p, u, z, y, x);\n  }\n  return s1 - s2;",
     "    for (int64_t x = 0; x <= i - 1; x++) s2 += val(p, u, z, y, x);\n  }\n  return s2 - s1;"),
    ("beta: far edge one column short", "P:327-332", "for (int64_t x = nx + i; x <= nx - 1; x++) s2 += val(p, u, z, y, x);",
     "for (int64_t x = nx + i + 1; x <= nx - 1; x++) s2 += val(p, u, z, y, x);"),
    ("a': ghost line of nx", "Theorem 1", "S = (double)ny * g;", "S = (double)nx * g;"),
    ("b': ghost line of ny", "Theorem 1", "S = (double)nx * g;", "S = (double)ny * g;"),
    ("a': dk sign", "Theorem 1, Q6", "int64_t zr = res(z + q->dk, nz, p->bc), xr = res(x + q->di, nx, p->bc);",
     "int64_t zr = res(z - q->dk, nz, p->bc), xr = res(x + q->di, nx, p->bc);"),
    ("a': di sign", "Theorem 1", "int64_t zr = res(z + q->dk, nz, p->bc), xr = res(x + q->di, nx, p->bc);",
     "int64_t zr = res(z + q->dk, nz, p->bc), xr = res(x - q->di, nx, p->bc);"),
    ("b': dj sign", "Theorem 1", "yr = res(y + q->dj, ny, p->bc);", "yr = res(y - q->dj, ny, p->bc);"),
    ("a': alpha at the unshifted column", "Q3", "if (q->dj != 0) S = S + alpha(p, u, zr, xr, q->dj);",
     "if (q->dj != 0) S = S + alpha(p, u, zr, x, q->dj);"),
    ("b': beta with dj", "Theorem 1", "if (q->di != 0) S = S + beta(p, u, zr, yr, q->di);",
     "if (q->di != 0) S = S + beta(p, u, zr, yr, q->dj);"),
    ("a': unrounded weight", "Q23", "        double w = rnd(p->dtype, q->w);\n        int64_t zr = res(z + q->dk, nz, p->bc), xr",
     "        double w = q->w;\n        int64_t zr = res(z + q->dk, nz, p->bc), xr"),
    ("a': c_x dropped", "Theorem 1", "double acc = cA[z * nx + x];", "double acc = 0.0;"),
    ("flag: absolute difference", "P:505-509", "double rel = fabs(pred / act - 1.0);", "double rel = fabs(pred - act);"),
    ("flag: 0 == 0 flagged", "Q24", "if (pred == act) return 0;", ""),
    ("flag: NaN passes", "Q24", "return !(rel <= eps);", "return rel > eps;"),
    ("locate: last flagged row", "P:232-234", "if (or_flag(PB[z * ny + y], B[z * ny + y], p->eps)) { if (y0 < 0) y0 = y; nb++; }",
     "if (or_flag(PB[z * ny + y], B[z * ny + y], p->eps)) { y0 = y; nb++; }"),
    ("lazy: skip on a instead of b", "P:496-497", "if (p->checksums == 1 && nb == 0) return 0;",
     "if (p->checksums == 1 && nb != 0) return 0;"),
    ("Eq. 8: vx alone", "P:642-657", "cor = p->correction_form == 2 ? cell_update(p, uprev, z, y0, x0) : rnd(p->dtype, (vx + vy) / 2.0);",
     "cor = p->correction_form == 2 ? cell_update(p, uprev, z, y0, x0) : rnd(p->dtype, vx);"),
    ("repair: a without the cell", "P:654", "A[z * nx + x0] = sx + cor;", "A[z * nx + x0] = sx;"),
    ("form 1: repair adds the value", "P:670-677", "A[z * nx + x0] += cor - uo;", "A[z * nx + x0] += cor;"),
    ("form 1: vy from a", "P:670-677", "vy = PB[z * ny + y0] - (B[z * ny + y0] - uo);", "vy = PB[z * ny + y0] - (A[z * nx + x0] - uo);"),
    ("form 2: recompute from u^s", "P:743-745, Q27", "const double v = cell_update(p, uprev, z, y, x);",
     "const double v = cell_update(p, u, z, y, x);"),
    ("status: unlocated / uncorrectable swapped", "Q13, Q14", "if (na == 0 || nb == 0) {\n    r.status = OR_REC_UNLOCATED;",
     "if (na != 0 && nb != 0) {\n    r.status = OR_REC_UNLOCATED;"),
    ("lazy: a from u^s", "P:271-273", "or_checksums(p, cur, Ap, Bt);", "or_checksums(p, nxt, Ap, Bt);"),
    ("online: alpha/beta from u^s", "Theorem 1", "or_predict(p, Ap, Bp, cur, cA, cB, PA, PB);",
     "or_predict(p, Ap, Bp, nxt, cA, cB, PA, PB);"),
    ("offline: prediction from u^t", "P:713-726", "or_predict(p, PA, PB, cur, cA, cB, QA, QB);",
     "or_predict(p, PA, PB, nxt, cA, cB, QA, QB);"),
    ("offline: no rollback", "P:696-698", "if (cur != ckpt) memcpy(cur, ckpt, fb);", ""),
    ("offline: record at window start", "P:737-745", "r.sweep = wend; r.z = z;", "r.sweep = s; r.z = z;"),
    ("partial: reach L - 1", "Q28", "const int64_t r = 2 * (wend - s - 1);", "const int64_t r = (wend - s - 1);"),
    ("partial: no periodic wrap", "Q28", "if (p->bc == OR_BC_PERIODIC && wraps) memset(redo, 1, (size_t)nz);", ""),
    ("partial: one interval over all flagged layers", "Q28", "memset(redo, 0, (size_t)nz);\n            for (int64_t f = 0;",
     "memset(redo, 0, (size_t)nz);\n            { int64_t f0 = nz, f1 = -1; for (int64_t f = 0; f < nz; f++) if (flagged[f]) { if (f < f0) f0 = f; f1 = f; }\n"
     "              for (int64_t z = f0; z <= f1; z++) redo[z] = 1; }\n            for (int64_t f = 0;"),
    # (re-checking every layer after a partial re-execution is an equivalent
    # mutant: the kept layers hold the values and predictions that did not
    # flag the first time)
    ("partial: first execution kept everywhere", "Q28", "if (!redo[z]) memcpy((char*)cur", "if (1) memcpy((char*)cur"),
    ("offline lazy: a compared", "Q29", "if (p->checksums != 1)\n            for (int64_t x = 0;", "if (1)\n            for (int64_t x = 0;"),
    ("offline: rollbacks not counted", "P:737", "stats->rollbacks++;", ";"),
]


def run(tests: list[str]) -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--all-cpu", action="store_true", help="survivors: run the whole -m 'not gpu' suite")
    a = ap.parse_args()
    work = tempfile.mkdtemp(prefix="oracle_mut_")
    for d in ("oracle", "tests", "abft_inputs"):
        shutil.copytree(os.path.join(ROOT, d), os.path.join(work, d),
                        ignore=shutil.ignore_patterns("__pycache__", "*.so"))
    shutil.copy(os.path.join(ROOT, "pytest.ini"), work)
    src = os.path.join(work, "oracle", "abft_oracle.c")
    with open(src) as f:
        orig = f.read()
    lines = []
    survivors = 0
    for name, cite, old, new in MUTANTS:
        if orig.count(old) != 1:
            lines.append(f"SKIP  {name}: pattern occurs {orig.count(old)} times")
            continue
        with open(src, "w") as f:
            f.write(orig.replace(old, new))
        b = subprocess.run(["make", "-s", "-B", "-C", os.path.join(work, "oracle")], capture_output=True, text=True)
        if b.returncode != 0:
            lines.append(f"BUILD {name}: {b.stderr.strip()[:200]}")
            continue
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                            *tests], cwd=work, capture_output=True, text=True)
        failed = [l for l in r.stdout.splitlines() if l.startswith("FAILED") or l.startswith("ERROR")]
        if r.returncode == 0:
            survivors += 1
            lines.append(f"ALIVE {name} ({cite})")
        else:
            first = failed[0].split(" - ")[0] if failed else f"rc={r.returncode}"
            lines.append(f"dead  {name} ({cite}) -- {first}")
        print(lines[-1], flush=True)
    with open(src, "w") as f:
        f.write(orig)
    shutil.rmtree(work, ignore_errors=True)
    summary = f"{len(MUTANTS)} mutants, {survivors} alive"
    print(summary)
    if a.out:
        with open(a.out, "w") as f:
            f.write("# tools/oracle_mutants.py: one mutation of oracle/abft_oracle.c at a time "
                    f"against {' '.join(tests)}\n")
            f.write("\n".join(lines) + "\n" + summary + "\n")


if __name__ == "__main__":
    run(["tests/test_oracle_pins.py"])
