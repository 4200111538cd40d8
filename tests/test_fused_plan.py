"""Host logic of the fused Ax+dssum schedule (GatherScatter.fused_plan), on CPU.

The plan is checked structurally (every shared gid exactly once, dependencies
only on Ax chunks scheduled earlier) and by emulating the kernel's dssum blocks
in numpy against the reference gather-scatter sums from the golden maps.
"""
import numpy as np
import pytest
import torch


def _gs(golden_spaces, key):
    from paper_2207_07098_b200.space import GatherScatter

    gid = torch.from_numpy(golden_spaces[f"{key}_gid"].astype(np.int64))
    perm = torch.from_numpy(golden_spaces[f"{key}_perm"].astype(np.int64))
    off = torch.from_numpy(golden_spaces[f"{key}_offsets"].astype(np.int64))
    E = int(golden_spaces[f"{key}_elements"].shape[0])
    nnn = gid.numel() // E
    n = round(nnn ** (1.0 / 3.0))
    return GatherScatter(gid, perm, off, (E, n, n, n)), E, nnn


def _decode(pl):
    a = pl.plan.numpy()
    m = pl.meta
    nb, cp, K = int(m[0]), int(m[1]), int(m[2])
    sched = a[m[3]:m[3] + nb]
    ndb = int((sched < 0).sum())
    dtab = a[m[4]:m[4] + 4 * ndb].reshape(ndb, 4)
    need = a[m[5]:m[5] + K]
    lo = a[m[6]:m[6] + K]
    return a, m, sched, dtab, need, lo, cp, K


@pytest.mark.parametrize("key,masked", [("pbox543", False), ("pbox543", True), ("pbox322", False),
                                        ("rotor", False), ("rotor", True)])
@pytest.mark.parametrize("chunk_pairs,lag", [(1, 1), (2, 1), (5, 1), (2, 3)])
def test_fused_plan_schedule(golden_spaces, key, masked, chunk_pairs, lag):
    gs, E, nnn = _gs(golden_spaces, key)
    rng = np.random.default_rng(7)
    perm = None
    keep = None
    if masked:
        keep = torch.from_numpy(rng.random(gs.P) > 0.2)
        perm = gs.masked_perm(keep)
    pl = gs.fused_plan(perm, chunk_pairs=chunk_pairs, lag=lag)
    a, m, sched, dtab, need, lo, cp, K = _decode(pl)
    npairs = (E + 1) // 2
    assert K == (npairs + cp - 1) // cp
    # every Ax pair exactly once; need[] matches
    apos = {int(j): t for t, j in enumerate(sched) if j >= 0}
    assert sorted(apos) == list(range(npairs))
    assert [sum(1 for j in apos if j // cp == k) for k in range(K)] == list(need)

    n2, n4, n8 = gs.cls_n
    p2 = a[m[7]:m[7] + 2 * n2].reshape(-1, 2)
    p4 = a[m[8]:m[8] + 4 * n4].reshape(-1, 4)
    p8 = a[m[9]:m[9] + 8 * n8].reshape(-1, 8)
    goff = a[m[10]:m[10] + gs.cls_n_gen + 1]
    gperm = a[m[11]:m[11] + int(goff[-1])]

    def items(d):
        k, cls, s, c = (int(x) for x in d)
        if cls == 2:
            return [p2[i] for i in range(s, s + c)]
        if cls == 4:
            return [p4[i] for i in range(s, s + c)]
        if cls == 8:
            return [p8[i] for i in range(s, s + c)]
        return [gperm[goff[i]:goff[i + 1]] for i in range(s, s + c)]

    # dependencies: a dssum block only reads elements of chunks lo[k]..k, all of
    # whose Ax pairs are scheduled before it
    seen = []
    for t, j in enumerate(sched):
        if j >= 0:
            continue
        d = dtab[-1 - j]
        k = int(d[0])
        for it in items(d):
            el = (it & 0x7FFFFFFF) // nnn
            ch = el // (2 * cp)
            assert lo[k] <= ch.min() and ch.max() == k
            seen.append(tuple(int(x) for x in it))
        for c in range(lo[k], k + 1):
            assert all(apos[p] < t for p in range(c * cp, min((c + 1) * cp, npairs)))
    ref_items = []
    cls_perm = (gs.cls_perm if perm is None else perm).numpy()
    o = 0
    for c, n in ((2, n2), (4, n4), (8, n8)):
        ref_items += [tuple(int(x) for x in r) for r in cls_perm[o:o + c * n].reshape(-1, c)]
        o += c * n + (gs.cls_pad2 if c == 2 else 0)
    go = gs.cls_gen_off.numpy()
    ref_items += [tuple(int(x) for x in cls_perm[o + go[i]:o + go[i + 1]]) for i in range(gs.cls_n_gen)]
    assert sorted(seen) == sorted(ref_items)

    # emulate the dssum blocks in schedule order and compare with the reference sums
    w = rng.standard_normal(gs.P)
    u = rng.standard_normal(gs.P)
    out = w.copy()
    for j in sched:
        if j < 0:
            for it in items(dtab[-1 - j]):
                s = 0.0
                for p in it:
                    s += w[p & 0x7FFFFFFF]
                for p in it:
                    out[p & 0x7FFFFFFF] = u[p & 0x7FFFFFFF] if p < 0 else s
    gid = golden_spaces[f"{key}_gid"]
    sums = np.zeros(int(gid.max()) + 1)
    for p in np.argsort(np.arange(gs.P), kind="stable"):
        sums[gid[p]] += w[p]
    want = sums[gid]
    if masked:
        km = keep.numpy()
        shared = np.bincount(gid)[gid] > 1
        want = np.where(shared & ~km, u, want)
    want = np.where(np.bincount(gid)[gid] > 1, want, w)
    assert np.array_equal(out, want)


@pytest.mark.parametrize("key", ["pbox543", "pbox322", "rotor", "cube222"])
def test_dssum_block_ranges(golden_spaces, key):
    """sf_dssum_blk_f64 schedule: per class, block b's items are exactly those whose
    lowest local copy lies in elements [b*eb, (b+1)*eb); every item once."""
    gs, E, nnn = _gs(golden_spaces, key)
    gs._build_classes()
    nb, eb = gs.cls_nb, gs.cls_eb
    bs = gs.cls_bstart.numpy().reshape(4, nb + 1)
    perm = gs.cls_perm.numpy()
    n2, n4, n8 = gs.cls_n
    go = gs.cls_gen_off.numpy()
    items = []
    o = 0
    for c, n in ((2, n2), (4, n4), (8, n8)):
        items.append([perm[o + c * i:o + c * (i + 1)] for i in range(n)])
        o += c * n + (gs.cls_pad2 if c == 2 else 0)
        assert c != 2 or o % 4 == 0        # quads start 16-byte aligned
    items.append([perm[o + go[i]:o + go[i + 1]] for i in range(gs.cls_n_gen)])
    assert nb * eb >= E
    for row, its in zip(bs, items):
        assert row[0] == 0 and row[-1] == len(its) and np.all(np.diff(row) >= 0)
        for b in range(nb):
            for it in its[row[b]:row[b + 1]]:
                assert b * eb <= it.min() // nnn < (b + 1) * eb
