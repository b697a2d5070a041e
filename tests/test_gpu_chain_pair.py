"""Split-bf16 fused chain on CTA pairs (csrc/mlp_chain_split.cuh mlp_chain_split_pair_kernel: 8-CTA
clusters of 256 rows, tcgen05.mma.cta_group::2 with each CTA supplying its rows of A and half of the
weight slice) against the single-CTA streamed form (the default: the pair form halves each SM's operand
reads and weight stream but the K-block ring is TMA-latency bound, so it measured no faster at cfg2 and
slower at cfg5, where 8-CTA clusters do not all fit at once): per element the same MMA
sequence, so predictions, penultimate activations and gradients are bit-identical."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ml():
    from paper_2201_05752_b200 import moseslab

    L = moseslab.lib()
    assert L.moses_device_check() == 0, L.moses_last_error()
    yield moseslab
    L.moses_debug_set_chain_pair(0)


def run(ml, pair, dims, p, x, y):
    L = ml.lib()
    L.moses_debug_set_chain_pair(pair)
    try:
        dm = ml.DeviceModel(p, ml.PREC_BF16X3, max(128, x.shape[0]))
        s = ml.predict(dm, x)
        h = ml.penultimate_activations(dm, x)
        g, loss = ml.gradients(dm, ml.RankingBatch(x, y), want_loss=True)
        dm.close()
    finally:
        L.moses_debug_set_chain_pair(0)
    return s, h, g, loss


@pytest.mark.parametrize("dims", [[164, 512, 512, 512, 512, 1], [16, 512, 512, 1], [512, 512, 512, 512, 1]])
@pytest.mark.parametrize("n", [1, 100, 300, 2560, 5000])
def test_pair_chain_bit_identical(ml, dims, n):
    p = ml.init_random(dims, 17, strict=False)
    rng = np.random.default_rng(n)
    x = rng.random((n, dims[0]))
    y = 0.1 + rng.random(n)
    a = run(ml, 1, dims, p, x, y)
    b = run(ml, 0, dims, p, x, y)
    for u, v in zip(a, b):
        assert np.array_equal(np.asarray(u), np.asarray(v))


def test_pair_chain_pooled_training_graph(ml):
    """The benched path (pooled training graph) with the pair chain: three steps, weights equal to the
    streamed form's bit for bit."""
    import torch

    L = ml.lib()
    dims = [164, 512, 512, 512, 512, 1]
    p = ml.init_random(dims, 12345, strict=False)
    off = ml.synth_offsets(1, 512 * 3, 8)
    probe = ml.DeviceModel(p, ml.PREC_BF16X3, 128)
    ld = probe.packed_ld
    probe.close()
    rows = int(off[-1])
    X = torch.empty((rows, ld), dtype=torch.float32, device="cuda")
    Y = torch.empty(512 * 3, dtype=torch.float32, device="cuda")
    assert L.moses_synth_features_device(1, 0, rows, 164, ml.DTYPE_F32, X.data_ptr(), ld) == 0
    assert L.moses_synth_labels_device(1, 0, 512 * 3, Y.data_ptr()) == 0
    OFF = torch.from_numpy(off).cuda()
    per = [int(off[(b + 1) * 512] - off[b * 512]) for b in range(3)]
    rows_pad = (max(per) + 127) // 128 * 128
    out = []
    for pair in (1, 0):
        L.moses_debug_set_chain_pair(pair)
        try:
            dm = ml.DeviceModel(p, ml.PREC_BF16X3, rows_pad)
            ml._ck(L.moses_train_graph_create_pooled(dm.h, X.data_ptr(), ld, Y.data_ptr(), OFF.data_ptr(), 3, 512,
                                                     rows_pad, 0.001, 0.9, 1))
            ml._ck(L.moses_train_graph_launch(dm.h, 3))
            out.append(dm.download().params)
            dm.close()
        finally:
            L.moses_debug_set_chain_pair(0)
    assert np.array_equal(out[0], out[1])
