"""The boundary (include/kge.h) on CPU: libkge.so loads without a GPU, exports every declared entry point, validates
configurations before touching the device, and the product package never imports the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "kge.h")).read()
    return sorted(set(re.findall(r"\b(kge_[a-z_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2004_08532_b200 import kge
    L = kge.lib()
    names = _declared()
    assert "kge_init" in names and "kge_train_step" in names and "kge_sample" in names and "kge_score" in names
    for n in names:
        assert hasattr(L, n), n


def test_config_default():
    from paper_2004_08532_b200 import kge
    c = kge._Config()
    kge.lib().kge_config_default(ctypes.byref(c))
    assert c.abi_version == 4 and c.neg_deg_k == 0 and c.neg_local == 0 and c.loss == 0 and c.dim == 400 and c.batch_size == 1024 and c.chunk_size == 256 and c.neg_k == 256


def _init_rc(**kw):
    from paper_2004_08532_b200 import kge
    c = kge._Config()
    kge.lib().kge_config_default(ctypes.byref(c))
    c.n_entities, c.n_relations = 100, 5
    for k, v in kw.items():
        setattr(c, k, v)
    h = np.zeros(4, np.int64)
    out = ctypes.c_void_p()
    rc = kge.lib().kge_init(ctypes.byref(out), ctypes.byref(c), h.ctypes.data_as(kge._i64p),
                            h.ctypes.data_as(kge._i64p), h.ctypes.data_as(kge._i64p), 4)
    return rc, kge.lib().kge_last_error().decode()


@pytest.mark.parametrize("kw,code", [
    (dict(chunk_size=300), -1),                # g does not divide B
    (dict(neg_k=0), -1),                       # k <= 0
    (dict(model=3, dim=12), -1),               # ComplEx needs d % 8 == 0
    (dict(dim=6), -1),                         # float4 rows
    (dict(abi_version=7), -1),
    (dict(n_entities=1 << 31), -2),            # ids must fit int32 on the device
    (dict(batch_size=8192, chunk_size=8, neg_k=256), -1),  # single-CTA dedup bound
    (dict(neg_local=2), -1),                   # a flag: 0 or 1 (ABI 3)
    (dict(neg_local=1, world_size=4, rank=0, n_entities=3), -1),  # local shards must be non-empty
])
def test_validation_before_device(kw, code):
    rc, msg = _init_rc(**kw)
    assert rc == code, msg
    assert msg


def test_no_device_is_an_error_not_a_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    rc, msg = _init_rc()
    assert rc == -4 and "CPU fallback" in msg


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2004_08532_b200")
    bad = re.compile(r"^\s*(import\s+oracle|from\s+oracle|from\s+\.\.oracle)|liboracle|\borc_[a-z]+\s*\(|oracle\.h", re.M)
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                s = open(os.path.join(dp, f)).read()
                assert not bad.search(s), f
    import subprocess
    from paper_2004_08532_b200.build import LIB
    syms = subprocess.run(["nm", "-D", LIB], capture_output=True, text=True).stdout
    assert "orc_" not in syms and "synth_" not in syms
