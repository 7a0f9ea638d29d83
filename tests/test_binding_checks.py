"""Host-side argument checks of the ctypes binding (no GPU: the library loads, no compute)."""
import numpy as np
import pytest

import paper_1811_05335_b200 as P


def _fake_plan(prec="c128", N=10, Mtot=8, device=0):
    p = P.Plan.__new__(P.Plan)
    p.prec = P.INFT_C128 if prec == "c128" else P.INFT_C64
    p.N, p.Mtot, p.device, p.d = N, Mtot, device, 1
    p._h = None
    return p


def test_buffer_checks():
    p = _fake_plan()
    p._check_buf(np.zeros((3, 10), np.complex128), 10, "f")
    p._check_buf(np.zeros(10, np.complex128), 10, "f")
    with pytest.raises(TypeError):
        p._check_buf(np.zeros((3, 10), np.complex64), 10, "f")
    with pytest.raises(ValueError):
        p._check_buf(np.zeros((3, 9), np.complex128), 10, "f")
    with pytest.raises(ValueError):
        p._check_buf(np.zeros((2, 8), np.complex128), 8, "out", R=3)
    with pytest.raises(ValueError):
        p._check_buf(np.zeros((2, 2, 10), np.complex128), 10, "f")
    p64 = _fake_plan("c64")
    p64._check_buf(np.zeros((3, 10), np.complex64), 10, "f")
    with pytest.raises(TypeError):
        p64._check_buf(np.zeros((3, 10), np.complex128), 10, "f")


def test_torch_dtype_names():
    torch = pytest.importorskip("torch")
    p = _fake_plan()
    p._check_buf(torch.zeros(3, 10, dtype=torch.complex128), 10, "f")
    with pytest.raises(TypeError):
        p._check_buf(torch.zeros(3, 10, dtype=torch.float64), 10, "f")


def test_node_shape_checks():
    P._check_nodes_shape(np.zeros(5), 1)
    P._check_nodes_shape(np.zeros((5, 1)), 1)
    P._check_nodes_shape(np.zeros((5, 2)), 2)
    with pytest.raises(ValueError):
        P._check_nodes_shape(np.zeros((5, 2)), 1)
    with pytest.raises(ValueError):
        P._check_nodes_shape(np.zeros(10), 2)
