"""The seeded workload generator: ResNet layouts match torchvision, streams are
reproducible, and the module holds no arithmetic of the method."""
import numpy as np
import pytest

import synth


@pytest.mark.parametrize("depth,n,tensors,bn_layers,bn_ch", [
    (50, 25_557_032, 161, 53, 26_560), (152, 60_192_808, 467, 155, 75_712)])
def test_resnet_layout(depth, n, tensors, bn_layers, bn_ch):
    sizes = synth.resnet_param_sizes(depth)
    assert sum(sizes) == n and len(sizes) == tensors
    ch = synth.resnet_bn_channels(depth)
    assert len(ch) == bn_layers and sum(ch) == bn_ch


def test_resnet_layout_matches_torchvision():
    tv = pytest.importorskip("torchvision")
    m = tv.models.resnet50()
    assert [p.numel() for p in m.parameters()] == synth.resnet_param_sizes(50)


def test_reproducible_and_structured():
    a = synth.grad_scale(1000)
    g1 = synth.grads(3, 5, 1000, a)
    g2 = synth.grads(3, 5, 1000, a)
    assert g1.dtype == np.float32 and np.array_equal(g1, g2)
    assert not np.array_equal(g1[0], g1[1])            # per-worker noise
    assert not np.array_equal(g1, synth.grads(3, 6, 1000, a))
    assert 1e-5 <= a.min() and a.max() <= 1e-1


def test_no_method_arithmetic_imported():
    import ast, inspect
    tree = ast.parse(inspect.getsource(synth))
    names = {a.name for n in ast.walk(tree) if isinstance(n, (ast.Import, ast.ImportFrom)) for a in n.names}
    mods = {n.module for n in ast.walk(tree) if isinstance(n, ast.ImportFrom)}
    assert not ({"oracle", "paper_1711_04325_b200"} & (names | mods))
