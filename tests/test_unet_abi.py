"""CPU tests of the U-Net C-ABI boundary (include/unet.h, NEXT-4): every declared symbol is exported,
the params struct and blob size agree with the seeded generator's parameter table, and without a
GPU the create call fails with a status code (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

from paper_2312_05410_b200 import pf, synth, unet

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "unet.h")


@pytest.fixture(scope="module")
def L():
    from paper_2312_05410_b200 import build
    build.build()
    return unet.lib()


def test_exports_every_declared_symbol(L):
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    names = sorted(set(re.findall(r"\b(un_[a-z_0-9]+)\s*\(", src)))
    assert {"un_create", "un_forward", "un_forward_device", "un_conv3x3", "un_rollout", "un_free"} <= set(names)
    for n in names:
        assert hasattr(L, n), n


@pytest.mark.parametrize("lb,widths", [(3, (16, 32, 64, 128)), (1, (16, 16, 32, 32)), (5, (32, 64, 64, 128))])
def test_blob_size_matches_parameter_table(L, lb, widths):
    p = unet.default_params(lb=lb, widths=widths)
    assert unet.blob_size(p) == synth.blob_size(lb, widths)


def test_defaults():
    p = unet.default_params()
    assert (p.abi_version, p.lb, tuple(p.widths), p.height, p.width) == (1, 3, (16, 32, 64, 128), 256, 256)


def test_create_without_gpu_fails_loudly(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(pf.PfError):
        unet.UNet(unet.default_params(height=32, width=32, max_batch=1))


def test_bad_params_rejected(L):
    for kw in (dict(height=12), dict(widths=(16, 24, 64, 128)), dict(lb=0), dict(max_batch=0)):
        with pytest.raises(pf.PfError):
            unet.UNet(unet.default_params(**kw))
