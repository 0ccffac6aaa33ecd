"""The reference arm's input generator (oracle/gen_torch.py: pure torch, no
libhbk) reproduces the product's benchmark tensors bit for bit, so the CPU
arm times the reference algorithm on exactly the tensor the GPU arm
measures."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_config_tables_agree():
    from oracle import gen_torch as G
    from paper_1904_03329_b200.generate import CONFIGS

    assert G.CONFIGS == CONFIGS


@pytest.mark.parametrize("config,scale", [("nell-2", 1.0), ("flickr-3d", 0.2),
                                          ("delicious-3d", 0.2), ("nell-1", 0.2), ("config1", 1.0)])
def test_torch_generator_matches_product(config, scale):
    from oracle import gen_torch as G
    from paper_1904_03329_b200.generate import config_tensor

    t = config_tensor(config, scale=scale)
    gi, gv = G.config_tensor(config, scale=scale)
    assert gi.shape[0] == t.nnz
    assert np.array_equal(gi.cpu().numpy().view(np.uint32), t.indices)
    assert np.array_equal(gv.cpu().numpy().view(np.int64), t.values.view(np.int64))
