"""Host tile plan of the config-3 CTA panel (riccati_cta.cu, plan_tiles): which
warp owns which 8x8 tile of the extended panel, in which list order. CPU test
through the library's debug export (not part of the C ABI)."""
import ctypes

import numpy as np

from paper_2512_09058_b200 import _lib


def _plan():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    lists = np.zeros(16 * 32, np.uint16)
    counts = np.zeros(16 * 16, np.uint8)
    nown = np.zeros(16, np.int32)
    dims = np.zeros(6, np.int32)
    rc = lib.cyqb_debug_cta_plan(lists.ctypes.data_as(ctypes.c_void_p), counts.ctypes.data_as(ctypes.c_void_p),
                                 nown.ctypes.data_as(ctypes.c_void_p), dims.ctypes.data_as(ctypes.c_void_p))
    assert rc == 0
    TT, CT, RT, MAXL, NPS, NW = (int(v) for v in dims)
    tiles = [[(int(e) >> 8, int(e) & 255) for e in lists[w * 32: w * 32 + nown[w]]] for w in range(NW)]
    return tiles, counts.reshape(16, 16), dict(TT=TT, CT=CT, RT=RT, MAXL=MAXL, NPS=NPS, NW=NW)


def test_every_list_tile_is_owned_once():
    tiles, _, d = _plan()
    TT, CT = d["TT"], d["CT"]
    # the pivot warp's tiles: the pivot diagonal (t, t) and the tile left of it
    pivot = {(t, t) for t in range(CT)} | {(t, t - 1) for t in range(1, CT)}
    expect = {(i, j) for i in range(TT) for j in range(i + 1)} - pivot
    owned = [t for w in tiles for t in w]
    assert len(owned) == len(set(owned)) == len(expect)
    assert set(owned) == expect
    assert tiles[0] == []  # the pivot warp holds no list tile
    assert max(len(w) for w in tiles) <= d["MAXL"] <= 15  # 4-bit counts, 15 packed slots


def test_lists_are_column_descending_with_skip_mode_pure_tiles_first():
    tiles, _, d = _plan()
    CT, RT, NPS = d["CT"], d["RT"], d["NPS"]
    for w, lst in enumerate(tiles[1:], start=1):
        # slots 0 .. NPS-1: pure coupling tiles (rows and columns all coupling rows)
        for ti, tj in lst[:NPS]:
            assert CT <= tj <= ti < RT, (w, ti, tj)
        cols = [tj for _, tj in lst[NPS:]]
        assert cols == sorted(cols, reverse=True), (w, cols)
        # the update prefix property: every tile with column > kb precedes every other
        for kb in range(CT):
            active = [tj > kb for _, tj in lst]
            assert active == sorted(active, reverse=True), (w, kb)


def test_counts_are_the_prefix_lengths():
    tiles, counts, d = _plan()
    for w, lst in enumerate(tiles):
        assert counts[w][0] == len(lst)
        for kb in range(d["CT"]):
            assert counts[w][kb + 1] == sum(tj > kb for _, tj in lst), (w, kb)


def test_the_pivot_warps_sub_partition_holds_only_the_first_block_columns():
    tiles, _, d = _plan()
    NPS = d["NPS"]
    for w in range(4, d["NW"], 4):
        assert all(tj <= 1 for _, tj in tiles[w][NPS:]), tiles[w]
    # and they are full, so that (almost) every tile of block columns 0 and 1 is
    # theirs: the bulk warps' first solves are of block column 2
    assert all(len(tiles[w]) == d["MAXL"] for w in range(4, d["NW"], 4))
    low = [(ti, tj) for w in range(d["NW"]) if w % 4 for ti, tj in tiles[w] if tj <= 1]
    assert len(low) <= 1, low
