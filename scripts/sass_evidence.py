#!/usr/bin/env python
"""Which Blackwell (sm_100a) features the built kernels use, from their SASS
(cuobjdump of paper_1901_06535_b200/librd.so; no GPU needed). Writes
profiles/<round>_sass_evidence.json: per kernel family, the count of each
tell-tale mnemonic (B200_PROFILING.md "What proves a Blackwell-native kernel")
and the registers / shared memory of the default instantiations.

  python scripts/sass_evidence.py --round r01
"""
import argparse
import collections
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1901_06535_b200", "librd.so")

MNEMONICS = {
    "UTMALDG": "TMA tensor load (cp.async.bulk.tensor)",
    "UBLKCP": "TMA 1-D bulk copy (cp.async.bulk)",
    "SYNCS.ARRIVE.TRANS64": "mbarrier arrive.expect_tx",
    "SYNCS.PHASECHK.TRANS64.TRYWAIT": "mbarrier try_wait.parity",
    "STAS": "st.async to a cluster peer's shared memory (DSMEM)",
    "UCGABAR_ARV": "cluster barrier arrive",
    "ELECT": "elect.sync (one issuing lane)",
    "MUFU.RCP": "fp32 reciprocal approximation (certified division)",
    "MUFU.RCP64H": "fp64 reciprocal approximation (inline div.rn fast path)",
    "CALL.REL.NOINC": "calls (out-of-line paths)",
    "STL": "local-memory stores (spills)",
    "HMMA": "legacy tensor-core MMA (not expected: no contraction)",
}
FAMILIES = ("tb_kernel", "lp_kernel", "cr_kernel", "mirror_kernel", "probe_kernel", "stamp_kernel",
            "divcert_kernel", "phi_index_kernel")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    per = collections.defaultdict(collections.Counter)
    kernels = collections.Counter()
    fam = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fam = next((f for f in FAMILIES if f in m.group(1)), None)
            if fam:
                kernels[fam] += 1
            continue
        if fam is None:
            continue
        ins = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if ins:
            op = ins.group(1)
            for mn in MNEMONICS:
                if op == mn or op.startswith(mn + "."):
                    per[fam][mn] += 1
    res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    usage = {}
    for want in ("tb_kernelIfLi4ELi4ELb1ELi4E", "cr_kernelIfLb1ELi4ELi768ELb0ELb1E", "cr_kernelIdLb1ELi2ELi768ELb1ELb1E",
                 "tb_kernelIdLi4ELi2ELb1ELi2E"):
        m = re.search(r"Function (\S*" + want + r"\S*):\s*\n\s*(REG:\d+.*)", res)
        if m:
            usage[m.group(1)] = m.group(2).strip()
    out = {"source": "cuobjdump -sass / -res-usage of librd.so (sm_100a)", "instantiations": dict(kernels),
           "mnemonics": {f: dict(c) for f, c in per.items()}, "legend": MNEMONICS, "resource_usage": usage}
    path = os.path.join(ROOT, "profiles", f"{a.round}_sass_evidence.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    for f in FAMILIES:
        if f in per:
            print(f"{f:18s} x{kernels[f]:3d}  " + ", ".join(f"{k}={v}" for k, v in sorted(per[f].items())))
    for k, v in usage.items():
        print(k[:60], v)


if __name__ == "__main__":
    main()
