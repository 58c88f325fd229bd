"""Host side of PM_LABELS_RUNS (include/pmap.h pm_label_runs): the binding's
encoder against a direct numpy decode of the documented word layout.  No GPU
(the device decode is checked against dense labels in test_gpu_parity.py)."""
import numpy as np
import pytest
import torch

pm = pytest.importorskip("paper_2411_01919_b200")


def _decode(runs, B, H, W):
    rs = runs.row_start.numpy().view(np.uint32).astype(np.int64)
    rr = runs.runs.numpy().view(np.uint32).astype(np.int64)
    assert rs.shape == (B * H + 1,) and rs[0] == 0 and np.all(np.diff(rs) >= 1)
    out = np.full((B * H, W), -1, np.int64)
    for g in range(B * H):
        x = 0
        for w in rr[rs[g]:rs[g + 1]]:
            lab, n = w & 0xFFFF, w >> 16
            assert n >= 1
            out[g, x:x + n] = -1 if lab == 0xFFFF else lab
            x += n
        assert x == W                       # the encoder covers each row exactly
    return out.reshape(B, H, W)


@pytest.mark.parametrize("seed", range(4))
def test_encode_label_runs_round_trip(seed):
    rng = np.random.default_rng(seed)
    B, H, W = 3, 17, 53
    lab = rng.integers(-3, 40, (B, H, W))
    lab[0] = 7                              # constant frame: one run per row
    lab[1, :, 20:] = -1                     # unlabelled tails
    lab[2, 5] = np.arange(W) % 2            # alternating: one run per pixel
    lab[2, 6, :3] = 0xFFFF + 5              # out-of-range labels read as none
    runs = pm.encode_label_runs(torch.from_numpy(lab.astype(np.int32)))
    want = np.where((lab < 0) | (lab >= 0xFFFF), -1, lab)
    assert np.array_equal(_decode(runs, B, H, W), want)
    rs = runs.row_start.numpy().view(np.uint32)
    assert rs[H] - rs[0] == H               # frame 0: H rows of one run
    assert rs[2 * H + 6] - rs[2 * H + 5] == W
    assert runs.nbytes == 4 * (B * H + 1 + rs[-1])


def test_encode_label_runs_rejects_bad_shapes():
    with pytest.raises(pm.PMError):
        pm.encode_label_runs(torch.zeros(4, 5, dtype=torch.int32))
