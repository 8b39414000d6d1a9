"""Executes the reference-side ctypes binding of INTEGRATION.md verbatim
(the code block tagged ``[integration-stub]``) against the in-tree library,
and checks it against the fp64 dense product: the documented boundary is the
one that works (encode -> TB2 -> linear forward, workspace prefix zeroed)."""

import os
import re

import pytest
import torch

from conftest import REPO

pytestmark = pytest.mark.gpu


def _stub_source() -> str:
    text = open(os.path.join(REPO, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    stub = [b for b in blocks if "[integration-stub]" in b]
    assert len(stub) == 1, "INTEGRATION.md must hold exactly one [integration-stub] block"
    return stub[0]


def test_integration_stub_parses():
    compile(_stub_source(), "INTEGRATION.md", "exec")


@pytest.mark.parametrize("M,adapters", [(1, True), (16, True), (32, False), (300, True)])
def test_integration_stub_runs(M, adapters, monkeypatch):
    monkeypatch.setenv("SALR_B200_LIB", os.path.join(REPO, "paper_2601_16991_b200", "libsalr_b200.so"))
    ns = {}
    exec(compile(_stub_source(), "INTEGRATION.md", "exec"), ns)
    g = torch.Generator().manual_seed(M)
    K, N = 1024, 1536
    w = (torch.randn(K, N, generator=g) * 0.02).bfloat16().float()
    w[torch.rand(K, N, generator=g) < 0.5] = 0
    x = torch.randn(M, K, generator=g).bfloat16().float()
    a_cat = (torch.randn(K, 32, generator=g) / 32).bfloat16().float()
    b_cat = (torch.randn(32, N, generator=g) * 0.02).bfloat16().float()
    weight = ns["prepare_weight"](w.cuda())
    ad = ns["prepare_adapters"](a_cat.cuda(), b_cat.cuda(), N) if adapters else None
    ws = ns["make_workspace"](M, N, K, ad[2] if ad else 0)
    y = ns["linear_forward"](x.cuda(), weight, ad, ws)
    y2 = ns["linear_forward"](x.cuda(), weight, ad, ws)  # workspace reuse
    ref = x.double() @ w.double()
    if adapters:
        ref += (x.double() @ a_cat.double()) @ b_cat.double()
    rel = float((y.double().cpu() - ref).norm() / ref.norm())
    mabs = float((y.double().cpu() - ref).abs().max() / ref.abs().max())
    print(f"integration M={M} adapters={adapters}: rel_frob={rel:.3e} max_abs={mabs:.3e}")
    assert rel <= 5e-4 and mabs <= 2.5e-4
    assert torch.equal(y, y2)
