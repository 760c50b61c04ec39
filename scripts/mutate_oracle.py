"""Mutation check of the oracle's pins (CPU only).

Each mutant is one plausible mistake in the oracle's C source (a dropped
term, a wrong sign, index or boundary, a latch off by one step). It is
applied to a scratch copy of the tree (mut_tmp/, removed afterwards; the
real oracle is never edited), liborc.so is rebuilt there, and the pin suites
(tests/test_oracle_pins.py, tests/test_circuits_oracle.py) run with -x. A
mutant is caught when they fail. Prints one JSON line per mutant.

  python scripts/mutate_oracle.py [--only "name1,name2"]
"""
import json
import os
import shutil
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MUT = os.path.join(ROOT, "mut_tmp")
BODY, LIBC = "oracle_body.h", "rd_oracle.c"
MUTANTS = [
 ("r operands swapped", BODY, "T r = (u - c->q) / (u + c->q);", "T r = (u + c->q) / (u - c->q);"),
 ("phi sign", BODY, "w = w + phi;", "w = w - phi;"),
 ("u - u^2 reversed", BODY, "T R = u - uu;", "T R = uu - u;"),
 ("reaction term sign", BODY, "R = R - (w * r);", "R = R + (w * r);"),
 ("u^2 dropped to u", BODY, "T uu = u * u;", "T uu = u;"),
 ("f*v dropped", BODY, "T w = c->f * v;", "T w = v;"),
 ("1/eps dropped", BODY, "return R * c->inv_eps;", "return R;"),
 ("south clamp wrong", BODY, "int64_t is = i < H - 1 ? i + 1 : H - 1;", "int64_t is = i < H - 1 ? i + 1 : H - 2;"),
 ("west clamp wrong", BODY, "int64_t jw = j > 0 ? j - 1 : 0;", "int64_t jw = j > 0 ? j - 1 : 1;"),
 ("east index = west", BODY, "T E = u[i * W + je];", "T E = u[i * W + jw];"),
 ("4C -> 3C", BODY, "T four_c = (T)4 * C;", "T four_c = (T)3 * C;"),
 ("1/dx^2 -> 1/dx", BODY, "c.inv_dx2 = (T)(1.0 / (p->dx * p->dx));", "c.inv_dx2 = (T)(1.0 / p->dx);"),
 ("v' dt dropped", BODY, "vo[k] = v[k] + c.dt * dv;", "vo[k] = v[k] + dv;"),
 ("dv sign", BODY, "T dv = C - v[k];", "T dv = v[k] - C;"),
 ("diffusion dropped", BODY, "T rhs = Ru + diff;", "T rhs = Ru;"),
 ("probe max -> min", BODY, "if (u[i * W + j] > m) m = u[i * W + j];", "if (u[i * W + j] < m || m == -(T)INFINITY) m = u[i * W + j];"),
 ("disc boundary excluded", LIBC, "if (dy * dy + dx * dx > 4 * s->r * s->r) return 0;",
  "if (dy * dy + dx * dx >= 4 * s->r * s->r) return 0;"),
 ("half-disc diameter excluded", LIBC, "return dx * DX[d] + dy * DY[d] >= 0;", "return dx * DX[d] + dy * DY[d] > 0;"),
 ("half-disc direction flipped", LIBC, "static const int64_t DX[4] = {1, 0, -1, 0};",
  "static const int64_t DX[4] = {-1, 0, 1, 0};"),
 ("rect end inclusive", LIBC, "return i >= s->y0 && i < s->y1 && j >= s->x0 && j < s->x1;",
  "return i >= s->y0 && i <= s->y1 && j >= s->x0 && j < s->x1;"),
 ("phi mask inverted", BODY, "if ((s->flags & ORC_SHAPE_MASK_PHI) && !(phi[i * W + j] == mphi)) continue;",
  "if ((s->flags & ORC_SHAPE_MASK_PHI) && (phi[i * W + j] == mphi)) continue;"),
 ("events one step late", BODY, "if (events[e].at_step == s) FN(orc_stamp)", "if (events[e].at_step == s - 1) FN(orc_stamp)"),
 ("latch records step s", BODY, "if (m >= (double)(T)pr->threshold) first_fire[pi] = s + 1;",
  "if (m >= (double)(T)pr->threshold) first_fire[pi] = s;"),
 ("probe stride off by one", BODY, "if (pr->stride > 0 && (s + 1) % pr->stride == 0 && first_fire[pi] < 0) {",
  "if (pr->stride > 0 && s % pr->stride == 0 && first_fire[pi] < 0) {"),
 ("latch not sticky", BODY, "if (pr->stride > 0 && (s + 1) % pr->stride == 0 && first_fire[pi] < 0) {",
  "if (pr->stride > 0 && (s + 1) % pr->stride == 0) {"),
 ("threshold exclusive", BODY, "if (m >= (double)(T)pr->threshold) first_fire[pi] = s + 1;",
  "if (m > (double)(T)pr->threshold) first_fire[pi] = s + 1;"),
 ("timelapse keeps min", BODY, "if (u[k] > max_u[k]) max_u[k] = u[k];", "if (u[k] < max_u[k]) max_u[k] = u[k];"),
 ("rest state phi sign", LIBC, "    w = w + phi;", "    w = w - phi;"),
 ("fault step off by one", BODY, "fault->step = s + 1;", "fault->step = s;"),
 ("fault cell transposed", BODY, "fault->i = bad / W;\n        fault->j = bad % W;",
  "fault->i = bad % W;\n        fault->j = bad / W;"),
]


def main():
    only = None
    if len(sys.argv) > 2 and sys.argv[1] == "--only":  # --only "name1,name2"
        only = set(sys.argv[2].split(","))
    res = []
    for name, fname, old, new in MUTANTS:
        if only is not None and name not in only:
            continue
        src = open(os.path.join(ROOT, "oracle", fname)).read()
        assert src.count(old) == 1, name
        if os.path.exists(MUT): shutil.rmtree(MUT)
        os.makedirs(MUT)
        for d in ("oracle", "rdinputs", "tests", "paper_1901_06535_b200"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(MUT, d), ignore=shutil.ignore_patterns("__pycache__", "*.o"))
        for f in ("pytest.ini", "conftest.py", "setup.cfg", "pyproject.toml"):
            if os.path.exists(os.path.join(ROOT, f)): shutil.copy(os.path.join(ROOT, f), MUT)
        open(os.path.join(MUT, "oracle", fname), "w").write(src.replace(old, new))
        subprocess.run([sys.executable, "-c", "import oracle; oracle.build(force=True)"], cwd=MUT, check=True,
                       capture_output=True)
        t0 = time.time()
        p = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "tests/test_circuits_oracle.py",
                            "-x", "-q", "-p", "no:cacheprovider"], cwd=MUT, capture_output=True, text=True, timeout=900)
        failed = [l for l in p.stdout.splitlines() if l.startswith("FAILED")]
        res.append({"mutant": name, "caught": p.returncode != 0, "by": failed[0][7:80] if failed else None,
                    "secs": round(time.time() - t0, 1)})
        print(json.dumps(res[-1]), flush=True)
    shutil.rmtree(MUT)
    print(json.dumps({"mutants": len(res), "caught": sum(r["caught"] for r in res)}))


if __name__ == "__main__":
    main()
