"""Mutation check of the oracle pins (scratch; run from the repo root)."""
import os, shutil, subprocess, sys, json, time
ROOT = os.path.dirname(os.path.abspath(__file__))
MUT = os.path.join(ROOT, "mut_tmp")
MUTANTS = [
 ("r operands swapped", "T r = (u - c->q) / (u + c->q);", "T r = (u + c->q) / (u - c->q);"),
 ("phi sign", "w = w + phi;", "w = w - phi;"),
 ("u - u^2 reversed", "T R = u - uu;", "T R = uu - u;"),
 ("reaction term sign", "R = R - (w * r);", "R = R + (w * r);"),
 ("u^2 dropped to u", "T uu = u * u;", "T uu = u;"),
 ("f*v dropped", "T w = c->f * v;", "T w = v;"),
 ("1/eps dropped", "return R * c->inv_eps;", "return R;"),
 ("south clamp wrong", "int64_t is = i < H - 1 ? i + 1 : H - 1;", "int64_t is = i < H - 1 ? i + 1 : H - 2;"),
 ("west clamp wrong", "int64_t jw = j > 0 ? j - 1 : 0;", "int64_t jw = j > 0 ? j - 1 : 1;"),
 ("east index = west", "T E = u[i * W + je];", "T E = u[i * W + jw];"),
 ("4C -> 3C", "T four_c = (T)4 * C;", "T four_c = (T)3 * C;"),
 ("1/dx^2 -> 1/dx", "c.inv_dx2 = (T)(1.0 / (p->dx * p->dx));", "c.inv_dx2 = (T)(1.0 / p->dx);"),
 ("v' dt dropped", "vo[k] = v[k] + c.dt * dv;", "vo[k] = v[k] + dv;"),
 ("dv sign", "T dv = C - v[k];", "T dv = v[k] - C;"),
 ("diffusion dropped", "T rhs = Ru + diff;", "T rhs = Ru;"),
 ("probe max -> min", "if (u[i * W + j] > m) m = u[i * W + j];", "if (u[i * W + j] < m || m == -(T)INFINITY) m = u[i * W + j];"),
]
def main():
    src = open(os.path.join(ROOT, "oracle", "oracle_body.h")).read()
    res = []
    for name, old, new in MUTANTS:
        assert src.count(old) == 1, name
        if os.path.exists(MUT): shutil.rmtree(MUT)
        os.makedirs(MUT)
        for d in ("oracle", "rdinputs", "tests", "paper_1901_06535_b200"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(MUT, d), ignore=shutil.ignore_patterns("__pycache__", "*.o"))
        for f in ("pytest.ini", "conftest.py", "setup.cfg", "pyproject.toml"):
            if os.path.exists(os.path.join(ROOT, f)): shutil.copy(os.path.join(ROOT, f), MUT)
        open(os.path.join(MUT, "oracle", "oracle_body.h"), "w").write(src.replace(old, new))
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
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", "mutants.json"), "w"), indent=1)
main()
