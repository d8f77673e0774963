"""tcgen05 weight-streaming GEMM vs a plain fp64 reference of the same product
(weights from the oracle generator, activations as the bf16 hi/lo pair)."""
import numpy as np
import pytest

from oracle import fso
from synth.configs import SHAPES

pytestmark = pytest.mark.gpu


def _hilo(x):
    import torch
    t = torch.from_numpy(x.astype(np.float32))
    hi = t.to(torch.bfloat16).float()
    lo = (t - hi).to(torch.bfloat16).float()
    return (hi + lo).double().numpy()


@pytest.mark.parametrize("name,which,rows,max_seg", [("small", 1, 13, 16), ("7b_l2", 0, 13, 16),
                                                     ("7b_l2", 1, 13, 16), ("7b_l2", 3, 13, 16),
                                                     ("7b_l2", 0, 61, 64), ("7b_l2", 1, 61, 64),
                                                     ("7b_l2", 3, 29, 32)])
def test_gemm_matches_fp64(name, which, rows, max_seg):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2507_02620_b200 import flowspec as F
    shape = SHAPES[name]
    gp = F.Pipeline(shape, max_ctx=1024, max_seg=max_seg)
    gp.fs_load_random_weights(11)
    gp.fs_set_prefix([1, 2, 3])
    model = fso.Model(shape, 11)
    if which == 0:
        W = np.concatenate([model.tensor(fso.Q), model.tensor(fso.K), model.tensor(fso.V)])
    elif which == 1:
        W = model.tensor(fso.O)
    else:
        W = model.tensor(fso.DOWN)
    rng = np.random.default_rng(0)
    X = rng.standard_normal((rows, W.shape[1])).astype(np.float32)
    Y = gp.debug_gemm(0, which, X, W.shape[0])
    ref = _hilo(X) @ W.astype(np.float64).T
    err = np.abs(Y - ref)
    scale = np.sqrt((X.astype(np.float64) ** 2).sum(1, keepdims=True) * (W.astype(np.float64) ** 2).mean())
    rel = float((err / scale).max())
    print(f"{name} which={which}: max abs {err.max():.3e}  max err/scale {rel:.3e}")
    # fp32 accumulation over K terms: |err| <~ K * 2^-24 * scale-ish
    assert rel < 5e-5   # tensor-core fp32 accumulation (measured ~1.3e-5 at K=4096)
