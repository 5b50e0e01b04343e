"""Structure of the ConvNeXt-1D harness against the paper's model description (CPU only).

The harness is how the bench line's model-level number (images/s) is measured, so its
oriented layers must be the ones PAPER.md's "Model Instantiation" specifies:
  * ConvNeXt-T-1D stage widths (96, 192, 384, 768) and depths (3, 3, 9, 3) (Table model_size);
  * K per stage [31, 31, 27, 15];
  * D = 8 directions i * 180 / 8 per layer, contiguous channel groups;
  * layer-wise rotation: +90 degrees on alternate layers (reading R11: per block);
  * the depthwise 1D stem: four 1x5 depthwise layers, strides 2, 1, 2, 1.
No kernel runs here: the module only records its geometry until it is called on a GPU.
"""
import numpy as np
import pytest

from paper_2309_15812_b200 import convnext1d


def _layers(name):
    m = convnext1d.ConvNeXt1D(name, num_classes=10)
    return list(convnext1d.oriented_layers(m))


@pytest.mark.parametrize("name,dims,depths", [
    ("convnext_t_1d", (96, 192, 384, 768), (3, 3, 9, 3)),
    ("convnext_b_1d", (128, 256, 512, 1024), (3, 3, 27, 3)),
])
def test_stage_widths_depths_and_kernel_caps(name, dims, depths):
    L = _layers(name)
    stem, blocks = L[:4], L[4:]
    assert [l.K for l in stem] == [5, 5, 5, 5]
    assert [l.stride for l in stem] == [2, 1, 2, 1]
    assert len(blocks) == sum(depths)
    i = 0
    for C, n, K in zip(dims, depths, (31, 31, 27, 15)):
        for l in blocks[i:i + n]:
            assert (l.C, l.K, l.stride) == (C, K, 1)
        i += n


def test_block_angles_are_eight_directions_rotated_on_alternate_layers():
    blocks = _layers("convnext_t_1d")[4:]
    base = np.arange(8) * 180.0 / 8
    for j, l in enumerate(blocks):
        a = np.asarray(l.angles_deg, dtype=np.float64)
        assert a.shape == (l.C,)
        shift = 90.0 * (j % 2)
        want = np.sort(np.mod(base + shift, 180.0))
        assert np.allclose(np.unique(np.mod(a, 180.0)), want)
        # contiguous groups of C / 8 channels per direction
        g = a.reshape(8, l.C // 8)
        assert np.all(g == g[:, :1])
        # the D=8 set maps onto itself under +90 degrees, so the rotation shows in the
        # order: group i carries i * 22.5 + shift
        assert np.allclose(np.mod(g[:, 0], 180.0), np.mod(base + shift, 180.0))
