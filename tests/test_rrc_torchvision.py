"""The RandomResizedCrop / CenterCrop window samplers against torchvision's own
code, given the same uniform draws.

The product's sampler (`csrc/orders.cpp:rrc_window`, run inside the loader) is
bit-identical to the oracle's `or_rrc_window` on every GPU parity test; this
test pins the oracle one step further, to the published semantics north_star
names: torchvision `RandomResizedCrop.get_params` (FFCV's `get_random_crop`
is the same rule in numpy float64).  torchvision's function body is executed
unmodified; only the `torch` module it draws from is swapped for a shim that
hands out the bbox Rng stream (uniform = a + (b - a) * u, randint(0, n) =
below(n)) in float64, so any difference in control flow, rounding, bounds or
fallback shows up as a window mismatch.
"""

import ctypes
import math

import numpy as np
import pytest

from oracle import oracle as O

tvt = pytest.importorskip("torchvision.transforms.transforms")

MASK64 = (1 << 64) - 1


class _Stream:
    """The draws or_rrc_window makes, in its order (bbx_oracle.c: or_uniform / or_below)."""

    def __init__(self, state):
        self.rng = O.PyRng(state)

    def uniform(self):
        return (self.rng.next_u64() >> 11) * (1.0 / 9007199254740992.0)

    def below(self, n):
        return self.rng.below(n)


class _Scalar:
    def __init__(self, v):
        self.v = float(v)

    def item(self):
        return self.v

    def __float__(self):
        return self.v


class _Vec:
    def __init__(self, vals):
        self.vals = [float(v) for v in vals]

    def __getitem__(self, i):
        return _Scalar(self.vals[i])


class _TorchShim:
    """The subset of `torch` get_params touches, fed from one _Stream."""

    def __init__(self, stream):
        self.s = stream

    def tensor(self, vals):
        return _Vec(vals)

    def log(self, v):
        return _Vec([math.log(x) for x in v.vals])

    def exp(self, v):
        return _Scalar(math.exp(float(v)))

    def empty(self, n):
        shim = self

        class _E:
            def uniform_(self, a, b):
                a, b = float(a), float(b)
                return _Scalar(a + (b - a) * shim.s.uniform())
        return _E()

    def randint(self, lo, hi, size=None):
        assert lo == 0
        return _Scalar(self.s.below(int(hi)))


def _oracle_window(state, h, w, scale, ratio):
    st = ctypes.c_uint64(state)
    t, l, ch, cw = (ctypes.c_int() for _ in range(4))
    O.lib().or_rrc_window(ctypes.byref(st), h, w, (ctypes.c_double * 2)(*scale), (ctypes.c_double * 2)(*ratio),
                          ctypes.byref(t), ctypes.byref(l), ctypes.byref(ch), ctypes.byref(cw))
    return t.value, l.value, ch.value, cw.value, st.value


def _torchvision_window(monkeypatch, state, h, w, scale, ratio):
    import torch
    stream = _Stream(state)
    with monkeypatch.context() as m:
        m.setattr(tvt, "torch", _TorchShim(stream))
        img = torch.empty((3, h, w), dtype=torch.uint8)
        i, j, hh, ww = tvt.RandomResizedCrop.get_params(img, list(scale), list(ratio))
    return int(i), int(j), int(hh), int(ww), stream.rng.state


@pytest.mark.parametrize("scale,ratio", [
    ((0.08, 1.0), (3 / 4, 4 / 3)),     # torchvision / FFCV defaults (configs[2])
    ((0.35, 1.0), (3 / 4, 4 / 3)),
    ((0.9, 1.0), (0.2, 0.3)),          # forces the fallback branch on square images
    ((0.01, 0.02), (1.0, 1.0)),        # tiny windows
])
def test_rrc_window_matches_torchvision_get_params(monkeypatch, scale, ratio):
    rs = np.random.default_rng(7)
    fallbacks = 0
    for trial in range(400):
        h, w = int(rs.integers(1, 700)), int(rs.integers(1, 700))
        state = int(rs.integers(0, 1 << 63)) * 2 + 1
        got = _oracle_window(state, h, w, scale, ratio)
        want = _torchvision_window(monkeypatch, state, h, w, scale, ratio)
        assert got == want, (trial, h, w, got, want)
        t, l, ch, cw, _ = got
        assert 0 <= t and t + ch <= h and 0 <= l and l + cw <= w and ch >= 1 and cw >= 1
        fallbacks += (t, l) == ((h - ch) // 2, (w - cw) // 2)
    assert fallbacks > 0


def test_center_window_matches_ffcv_rule():
    """CenterCrop(ratio): side = int(ratio * min(h, w)), centred (FFCV get_center_crop);
    checked through the oracle's chain on the sampled window size."""
    rs = np.random.default_rng(3)
    field = {"kind": "image", "max_h": 96, "max_w": 96, "channels": 3}
    for trial in range(40):
        h, w = int(rs.integers(8, 90)), int(rs.integers(8, 90))
        img = rs.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        side = int(0.875 * min(h, w))
        # an output the size of the window is a pure crop: the window's pixels, unresampled
        out, _ = O.chain_one(O.parse_spec(f"center:{side},{side},0.875"), field, h, w, 3, 0, img.reshape(-1), 1)
        t, l = (h - side) // 2, (w - side) // 2
        assert np.array_equal(out.reshape(side, side, 3), img[t:t + side, l:l + side]), trial
