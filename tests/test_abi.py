"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol the header
declares, and rejects invalid problems with the same status codes as the oracle (validation runs
before any device work, so these calls never touch CUDA)."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import oracle
import paper_2511_15629_b200 as E
from helpers import to_oracle
import workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "esdp.h")).read()
    return sorted(set(re.findall(r"^\s*(?:esdp_status|void|const char\*)\s+(esdp_\w+)\s*\(", src, re.M)))


def test_header_symbols_exported():
    names = _declared()
    assert len(names) >= 15
    lib = ctypes.CDLL(E.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(E.EXPORTED_SYMBOLS) == names


def test_oracle_and_product_share_no_code():
    """The product sources never include or load the oracle, and vice versa."""
    for d, bad in [(os.path.join(ROOT, "paper_2511_15629_b200"), "oracle"), (os.path.join(ROOT, "oracle"), "paper_2511_15629_b200")]:
        for root, _, files in os.walk(d):
            for f in files:
                if f.endswith((".cu", ".cuh", ".c", ".h", ".py")):
                    txt = open(os.path.join(root, f)).read()
                    if bad == "oracle":
                        assert "esdp_oracle" not in txt and "liboracle" not in txt, f
                        assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                    else:
                        assert "import paper_2511_15629_b200" not in txt and "libesdp" not in txt, f
                        assert not re.search(r'#include\s*[<"].*esdp\.h', txt), f


def _create_status(inst):
    try:
        ctx = E.esdp_create(inst.T, inst.K, inst.pbar, inst.sbar, inst.s0, inst.eta_c, inst.eta_d, inst.delta,
                            inst.lam, inst.P, inst.pi, inst.actions, inst.payoff_kind, inst.g, 0)
    except E.EsdpError as e:
        return e.status
    E.esdp_destroy(ctx)
    return 0


def _bad_cases():
    base = workloads.cfg1("b")
    out = []
    def mk(**kw):
        inst = workloads.cfg1("b")
        for k, v in kw.items():
            setattr(inst, k, v)
        return inst
    out.append(mk(eta_c=0.0))
    out.append(mk(eta_d=1.2))
    out.append(mk(sbar=100.5))
    out.append(mk(delta=-1.0))
    out.append(mk(s0=150.0))
    out.append(mk(pbar=0.0))
    lam = base.lam.copy(); lam[3, 2] = np.inf
    out.append(mk(lam=lam))
    P = base.P.copy(); P[5, 1, 0] += 0.01
    out.append(mk(P=P))
    out.append(mk(pi=np.array([0.5, 0.5, 0.5, -0.5, 0.0])))
    out.append(mk(actions=np.array([-1.0, 0.5, 0.0])))
    out.append(mk(actions=np.array([-1.0, -0.5, 0.5])))
    out.append(mk(actions=np.array([-20.0, 0.0, 1.0])))
    out.append(mk(payoff_kind=workloads.PAYOFF_LINEAR_MINUS_G, g=None))
    return out


@pytest.mark.parametrize("j", range(13))
def test_invalid_inputs_match_oracle_status(j):
    inst = _bad_cases()[j]
    want = oracle.status_of(to_oracle(inst))
    assert want in (oracle.REF_E_CONFIG, oracle.REF_E_DATA)
    assert _create_status(inst) == want
    assert E.esdp_last_error(None)


def test_binding_has_no_fallback():
    """The binding exposes only the C ABI; there is no numpy/CPU compute path to fall back to."""
    src = open(os.path.join(ROOT, "paper_2511_15629_b200", "__init__.py")).read()
    assert "import torch" not in src and "oracle" not in src


def test_header_compiles_as_c_and_matches_binding_layout(tmp_path):
    """A plain C11 program compiles against include/esdp.h, links against libesdp.so taking the address of
    every declared entry point (no call, so no GPU), and prints the esdp_problem layout; the ctypes struct of
    the binding must have the same size and field offsets (the binding hand-declares it)."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    names = _declared()
    fields = [f for f, _ in E.esdp_problem._fields_]
    cfield = {"lambda_": "lambda"}
    src = ["#include <stdio.h>", "#include <stddef.h>", '#include "esdp.h"',
           "_Static_assert(sizeof(int32_t) == 4 && sizeof(double) == 8, \"LP64 ABI\");",
           "typedef void (*fn_t)(void);", "int main(void) {", "  const fn_t fns[] = {"]
    src += [f"    (fn_t)&{n}," for n in names]
    src += ["  };", "  int n = 0;", "  for (unsigned i = 0; i < sizeof fns / sizeof fns[0]; ++i) n += fns[i] != 0;",
            '  printf("%d %zu\\n", n, sizeof(esdp_problem));']
    src += [f'  printf("%zu\\n", offsetof(esdp_problem, {cfield.get(f, f)}));' for f in fields]
    src += ["  return 0;", "}"]
    c = tmp_path / "abi.c"
    c.write_text("\n".join(src) + "\n")
    exe = tmp_path / "abi"
    lib = os.path.dirname(E.LIB_PATH)
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-pedantic", "-I", os.path.join(ROOT, "include"), str(c),
                    "-o", str(exe), "-L", lib, "-l:libesdp.so", f"-Wl,-rpath,{lib}"], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    assert int(out[0]) == len(names)
    assert int(out[1]) == ctypes.sizeof(E.esdp_problem)
    assert [int(x) for x in out[2:]] == [getattr(E.esdp_problem, f).offset for f in fields]
