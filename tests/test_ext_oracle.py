"""Pinning of the schema-extension kinds' oracle (oracle/planc_oracle.py
eval_ext) against torch's float64 implementations — forward values and
autograd gradients. The reference has no softmax / layernorm / GELU
(document.cpp:43-53), so torch is the independent implementation these
restatements are checked against."""
import numpy as np
import pytest
import torch

from oracle import planc_oracle as po

F = torch.nn.functional


@pytest.mark.parametrize("rows,n,seg", [(6, 16, 4), (5, 32, 0), (3, 24, 8), (1, 7, 0)])
def test_softmax_and_grad_match_torch(rows, n, seg):
    rng = np.random.default_rng(rows * n)
    x = rng.standard_normal((rows, n)) * 3
    dy = rng.standard_normal((rows, n))
    s = seg or n
    xt = torch.tensor(x, requires_grad=True)
    yt = torch.softmax(xt.view(rows, n // s, s), dim=-1).view(rows, n)
    yt.backward(torch.tensor(dy))
    y = po.eval_ext("softmax", [x], seg)
    assert np.allclose(y, yt.detach().numpy(), rtol=0, atol=1e-15)
    dx = po.eval_ext("softmax-grad", [y, dy], seg)
    assert np.allclose(dx, xt.grad.numpy(), rtol=0, atol=1e-14)


@pytest.mark.parametrize("rows,n,seg,eps", [(6, 16, 0, 1e-5), (4, 64, 16, 1e-5), (3, 8, 0, 1e-3)])
def test_layernorm_and_grad_match_torch(rows, n, seg, eps):
    rng = np.random.default_rng(rows + n)
    x = rng.standard_normal((rows, n)) * 2 + 1
    dy = rng.standard_normal((rows, n))
    s = seg or n
    xt = torch.tensor(x, requires_grad=True)
    yt = F.layer_norm(xt.view(rows, n // s, s), (s,), eps=eps).view(rows, n)
    yt.backward(torch.tensor(dy))
    assert np.allclose(po.eval_ext("layernorm", [x], seg, eps), yt.detach().numpy(), rtol=0, atol=1e-13)
    assert np.allclose(po.eval_ext("layernorm-grad", [x, dy], seg, eps), xt.grad.numpy(), rtol=0, atol=1e-12)


def test_gelu_and_grad_match_torch():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((7, 9)) * 3
    dy = rng.standard_normal((7, 9))
    xt = torch.tensor(x, requires_grad=True)
    yt = F.gelu(xt)
    yt.backward(torch.tensor(dy))
    assert np.allclose(po.eval_ext("gelu", [x]), yt.detach().numpy(), rtol=0, atol=1e-14)
    assert np.allclose(po.eval_ext("gelu-grad", [x, dy]), xt.grad.numpy(), rtol=0, atol=1e-13)


def test_segment_alignment_is_enforced():
    with pytest.raises(po.UsageError):
        po.eval_ext("softmax", [np.zeros((2, 6))], 4)
    with pytest.raises(po.UsageError):
        po.eval_ext("softmax", [np.zeros((2, 8))], 4, in_masks=[{"region": [[0, 2], [2, 10]]}])


def test_attention_oracle_vs_torch():
    """The float64 attention restatement and its gradients against torch's
    scaled_dot_product_attention and autograd (causal and not)."""
    import numpy as np
    import torch

    from oracle import planc_oracle as po

    rng = np.random.default_rng(0)
    T, nh, dh, seq = 256, 2, 32, 128
    q, k, v, do = (rng.standard_normal((T, nh * dh)) for _ in range(4))
    sh = lambda x: x.reshape(T // seq, seq, nh, dh).transpose(0, 2, 1, 3)  # noqa: E731
    for causal in (False, True):
        o = po.attention(q, k, v, dh, seq, causal)
        tq, tk, tv = (torch.tensor(sh(x), requires_grad=True) for x in (q, k, v))
        out = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, is_causal=causal)
        assert np.abs(out.detach().numpy().transpose(0, 2, 1, 3).reshape(T, -1) - o).max() < 1e-12
        out.backward(torch.tensor(sh(do)))
        for w, t in (("q", tq), ("k", tk), ("v", tv)):
            g = po.attention_grad(q, k, v, o, do, dh, seq, causal, w)
            assert np.abs(g - t.grad.numpy().transpose(0, 2, 1, 3).reshape(T, -1)).max() < 1e-12, (causal, w)
