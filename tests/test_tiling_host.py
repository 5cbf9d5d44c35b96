"""Host logic of multi-ciphertext tiling (paper_2604_11659_b200/tiling.py):
grid choice, block split/reassembly, the block-product enumeration and the
work count (pairs over all block products == the untiled CSR x CSC schedule).
"""

import numpy as np
import pytest


def test_tile_grid_fits_slots():
    from paper_2604_11659_b200.tiling import tile_grid
    assert tile_grid(128, 32768) == (1, 128)             # cfg3 fits one ciphertext
    assert tile_grid(256, 32768) == (2, 128)             # configs[3] at N=2^16
    assert tile_grid(512, 65536) == (2, 256)             # configs[4] at N=2^17
    assert tile_grid(40, 512) == (2, 20)
    for n, slots in [(7, 16), (100, 512), (513, 4096)]:
        T, b = tile_grid(n, slots)
        assert b * b <= slots and T * b >= n
        assert T == 1 or (-(-n // (T - 1))) ** 2 > slots


def test_split_blocks_reassembles():
    from paper_2604_11659_b200 import formats
    from paper_2604_11659_b200.tiling import split_blocks
    m = formats.generate_random_sparse(37, 0.8, (5, 0))
    for T in (1, 2, 3, 4):
        blocks, b = split_blocks(m, T)
        full = np.zeros((T * b, T * b))
        for (I, K), blk in blocks.items():
            assert blk.shape == (b, b) and np.count_nonzero(blk)
            full[I * b:(I + 1) * b, K * b:(K + 1) * b] = blk
        assert np.array_equal(full[:37, :37], m)
        assert not full[37:, :].any() and not full[:, 37:].any()


@pytest.mark.parametrize("n,sp,T", [(24, 0.5, 2), (33, 0.9, 3), (64, 0.97, 4)])
def test_tiled_pairs_equal_untiled_schedule(n, sp, T):
    from paper_2604_11659_b200 import encmat, formats
    from paper_2604_11659_b200.tiling import tiled_pair_count
    a = formats.generate_random_sparse(n, sp, (11, 0))
    b = formats.generate_random_sparse(n, sp, (11, 1))
    ma, _ = encmat.meta_and_values(a, encmat.Layout.CSR)
    mb, _ = encmat.meta_and_values(b, encmat.Layout.CSC)
    assert tiled_pair_count(a, b, T) == len(encmat.pair_array(ma, mb))


def test_block_products_skip_empty_blocks():
    from paper_2604_11659_b200.encmat import Layout
    from paper_2604_11659_b200.tiling import TiledMatrix, block_products
    ta = TiledMatrix(n=4, T=2, b=2, layout=Layout.CSR, tiles={(0, 0): 1, (1, 1): 1})
    tb = TiledMatrix(n=4, T=2, b=2, layout=Layout.CSC, tiles={(0, 1): 1, (1, 0): 1, (1, 1): 1})
    assert block_products(ta, tb) == [(0, 0, 1), (1, 1, 0), (1, 1, 1)]
