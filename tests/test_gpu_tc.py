"""tcgen05 (5th-generation tensor core) 3xTF32 layer chains (hmdp_tc.cu) against an
FP64 reference of the same MLP (MlpT::forward, inference.cpp:87-101): the 3xTF32
split must stay at FP32 accuracy (single-pass TF32 would not)."""
import ctypes

import numpy as np
import pytest

import paper_2602_02234_b200 as P
from paper_2602_02234_b200._lib import check, lib, ptr

pytestmark = pytest.mark.gpu


def tc_mlp(x, layers):
    """layers: [(W [N][K], b [N], act)] -> y via hmdp_tc_mlp (FP32 in/out)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    sizes = np.array([x.shape[1]] + [W.shape[0] for W, _, _ in layers], dtype=np.int32)
    Wc = np.ascontiguousarray(np.concatenate([W.ravel() for W, _, _ in layers]), dtype=np.float32)
    bc = np.ascontiguousarray(np.concatenate([b for _, b, _ in layers]), dtype=np.float32)
    act = np.array([a for _, _, a in layers], dtype=np.int32)
    y = np.zeros((x.shape[0], sizes[-1]), dtype=np.float32)
    check(lib().hmdp_tc_mlp(0, x.shape[0], ptr(x), len(layers), ptr(sizes), ptr(Wc), ptr(bc),
                            ptr(act), ptr(y)))
    return y


def ref_mlp(x, layers):
    h = np.asarray(x, dtype=np.float32).astype(np.float64)
    for W, b, a in layers:
        h = h @ W.astype(np.float32).astype(np.float64).T + b.astype(np.float32)
        if a:
            h = np.tanh(h)
    return h


@pytest.mark.parametrize("rows", [1, 128, 300, 4114])
@pytest.mark.parametrize("shape", [(32, 64, 32, 32), (64, 32, 32), (16, 32, 32, 32), (8, 32)])
def test_tc_chain_fp32_accurate(rows, shape):
    rng = np.random.default_rng(rows + len(shape))
    layers = []
    for k, (K, N) in enumerate(zip(shape[:-1], shape[1:])):
        W = rng.normal(0, 1 / np.sqrt(K), (N, K))
        b = rng.normal(0, 0.1, N)
        layers.append((W, b, 1 if k < len(shape) - 2 else 0))
    x = rng.normal(0, 1.0, (rows, shape[0]))
    y = tc_mlp(x, layers)
    r = ref_mlp(x, layers)
    scale = max(1.0, float(np.abs(r).max()))
    err = float(np.abs(y - r).max()) / scale
    assert err < 3e-6, err  # FP32-level (single-pass TF32 would be ~1e-3)


def test_tc_embedding_chain_matches_model():
    """The DPA3 embedding + first message projection as one tcgen05 chain on a real
    model's weights: desc (16, zero-padded to 32) -> tanh(32) -> h0 (32) -> P0 (32)."""
    m = P.make_model(P.ModelFamily.message_passing, 3, 0.6, 2, 8, 32, 1).as_dict()
    e = m["embedding"]
    W1 = np.zeros((32, 32))
    W1[:, :16] = np.array(e["weights"][0]).reshape(32, 16)
    b1 = np.array(e["biases"][0])
    W2 = np.array(e["weights"][1]).reshape(32, 32)
    b2 = np.array(e["biases"][1])
    W1h = np.array(m["layers"][0]["message"]["weights"][0]).reshape(32, 40)[:, :32]
    layers = [(W1, b1, 1), (W2, b2, 0), (W1h, np.zeros(32), 0)]
    rng = np.random.default_rng(7)
    x = np.zeros((4114, 32))
    x[:, :16] = rng.uniform(0, 3, (4114, 16))  # descriptor-like magnitudes
    y = tc_mlp(x, layers)
    r = ref_mlp(x, layers)
    assert np.abs(y - r).max() < 3e-6 * max(1.0, np.abs(r).max())


def test_tcgen05_probe_positive():
    v = ctypes.c_double()
    check(lib().hmdp_peak_tcgen05_tf32(0, 50, ctypes.byref(v)))
    assert v.value > 100.0  # TFLOP/s, raw kind::tf32
