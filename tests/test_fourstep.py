"""Four-step split of one multiply: the host orchestration's data movement.

The device stages are replaced by a stand-in that tags every element with (polynomial,
global element index) and asserts, at every phase, that each element sits where the
layout of include/dkss.h says it must: columns [E][C] per rank, rows [R][mu0] after the
exchange, columns again after the way back, [E][mu0] after the gather.  Runs with the
emulated ranks in one process and over gloo with world size 2 (CPU).  The device stages
themselves are checked against a*b in tests/test_gpu_parity.py.
"""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_1503_04955_b200.fourstep import DistExchange, FourStepRank, run_rank, run_virtual

M, MM, LL = 64, 4, 2  # toy geometry: E = 8, mu0 = 16, element = 8 words
E, MU0, EW = 2 * MM, 2 * M // (2 * MM), MM * LL
A_TAG, B_TAG, PROD_TAG, SCALED_TAG = 1, 2, 7, 9


SEG = 5  # stand-in segment length of the distributed decode


class TagStages:
    def __init__(self, dist=False):
        self.calls = []
        self.dist = dist

    def layout(self, world):
        return {"cols": MU0 // world, "rows": E // world, "elem_words": EW, "block_words": 2 * M * EW // world,
                "decode_seg": SEG if self.dist else 0}

    def decode_partial(self, rank, world, x, s_out):
        # the columns must be the scaled product of exactly this rank's columns
        self.columns_seen(rank, world, x)
        v = s_out.view(E + 1, SEG)
        v[:, 0] = rank
        v[:, 1] = torch.arange(E + 1)
        self.calls.append("decode_partial")

    def columns_seen(self, rank, world, x):
        C = MU0 // world
        v = x.view(E, C, EW)
        want = torch.arange(E).view(E, 1) * MU0 + rank * C + torch.arange(C).view(1, C)
        assert bool((v[:, :, 0] == SCALED_TAG).all()) and torch.equal(v[:, :, 1], want.to(torch.int32))

    def decode_finish(self, world, parts, out):
        v = parts.view(world, E + 1, SEG)
        assert torch.equal(v[:, :, 0], torch.arange(world).view(world, 1).expand(world, E + 1).to(v.dtype))
        assert torch.equal(v[:, :, 1], torch.arange(E + 1).view(1, E + 1).expand(world, E + 1).to(v.dtype))
        out.fill_(1)
        self.calls.append("decode")

    def columns_fwd(self, rank, world, a, b, x):
        C = MU0 // world
        v = x.view(2, E, C, EW)
        v.zero_()
        for q, tag in enumerate((A_TAG, B_TAG)):
            v[q, :, :, 0] = tag
            j = torch.arange(E).view(E, 1)
            c = torch.arange(C).view(1, C)
            v[q, :, :, 1] = (j * MU0 + rank * C + c).to(torch.int32)
        self.calls.append("columns_fwd")

    def rows(self, rank, world, z):
        R = E // world
        v = z.view(2, R, MU0, EW)
        want = (torch.arange(R).view(R, 1) + rank * R) * MU0 + torch.arange(MU0).view(1, MU0)
        for q, tag in enumerate((A_TAG, B_TAG)):
            assert bool((v[q, :, :, 0] == tag).all()), "row phase got elements of the wrong polynomial"
            assert torch.equal(v[q, :, :, 1], want.to(torch.int32)), "row phase got misplaced elements"
        v[0, :, :, 0] = PROD_TAG
        self.calls.append("rows")

    def columns_inv(self, rank, world, x):
        C = MU0 // world
        v = x.view(E, C, EW)
        want = torch.arange(E).view(E, 1) * MU0 + rank * C + torch.arange(C).view(1, C)
        assert bool((v[:, :, 0] == PROD_TAG).all())
        assert torch.equal(v[:, :, 1], want.to(torch.int32))
        v[:, :, 0] = SCALED_TAG
        self.calls.append("columns_inv")

    def block_transpose(self, src, dst, n, A, B, run_words):
        dst.view(n, B, A, run_words).copy_(src.view(n, A, B, run_words).transpose(1, 2))

    def decode(self, v, out):
        w = v.view(2 * M, EW)
        assert bool((w[:, 0] == SCALED_TAG).all())
        assert torch.equal(w[:, 1], torch.arange(2 * M, dtype=torch.int32))
        out.fill_(1)
        self.calls.append("decode")


def _ranks(world, dist=False):
    st = TagStages(dist)
    return st, [FourStepRank(st, r, world, M, MM, torch.device("cpu"), 4) for r in range(world)]


@pytest.mark.parametrize("dist", [False, True])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_virtual_ranks_move_every_element(world, dist):
    st, ranks = _ranks(world, dist)
    a = torch.zeros(4, dtype=torch.int32)
    out = run_virtual(ranks, a, a)
    assert out.tolist() == [1, 1, 1, 1]
    assert st.calls.count("columns_fwd") == world and st.calls.count("rows") == world
    assert st.calls.count("columns_inv") == world and st.calls[-1] == "decode"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, distd=False):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        st = TagStages(distd)
        fs = FourStepRank(st, rank, world, M, MM, torch.device("cpu"), 4)
        a = torch.zeros(4, dtype=torch.int32)
        out = run_rank(fs, DistExchange(), a, a)
        q.put((rank, None if out is None else out.tolist(), st.calls, None))
    except Exception as e:  # report, do not hang the peer
        q.put((rank, None, [], repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
@pytest.mark.parametrize("distd", [False, True])
def test_two_rank_gloo_fourstep_exchange(distd):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, distd)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=150) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    for rank, out, calls, err in res:
        assert err is None, f"rank {rank}: {err}"
        assert calls[:3] == ["columns_fwd", "rows", "columns_inv"]
    assert res[0][1] == [1, 1, 1, 1] and res[0][2][-1] == "decode"
    assert res[1][1] is None


# --- the fused exchange (peer stores), CPU stand-in -----------------------------------------
# The device kernels store each output element at the address peer_dst() computes
# (csrc/dkss_kernels.cuh: out_elem / peer_dst).  The stand-in below restates that formula in
# Python and scatters tagged elements with it; TagStages then checks that every rank's rows and
# columns hold exactly the elements the all-to-all path delivers.

def peer_index(mode, world, rank, q_or_row, pos):
    """(destination rank, element index) of output element `pos` of launch polynomial
    `q_or_row` -- the Python restatement of csrc/dkss_kernels.cuh peer_dst()."""
    C, R = MU0 // world, E // world
    if mode == 1:  # columns [2][E][C] -> rows [2][R][MU0]
        j, c = pos // C, pos % C
        return j // R, (q_or_row * R + j % R) * MU0 + rank * C + c
    return pos // C, (rank * R + q_or_row) * C + pos % C  # rows [R][MU0] -> columns [E][C]


class TagPeerStages(TagStages):
    """TagStages with the fused-exchange entry points (peer tables map data_ptr -> tensor)."""

    def __init__(self):
        super().__init__(dist=True)
        self.by_ptr = {}

    def register(self, ranks):
        for fs in ranks:
            for t in (fs.z, fs.x, fs.gath):
                self.by_ptr[t.data_ptr()] = t

    def columns_fwd_peer(self, rank, world, a, b, x, z_peers):
        self.columns_fwd(rank, world, a, b, x)  # the tagged outputs of this rank's columns
        C = MU0 // world
        xv = x.view(2, E * C, EW)
        dst = [self.by_ptr[p].view(-1, EW) for p in z_peers.tolist()]
        for q in range(2):
            for pos in range(E * C):
                h, i = peer_index(1, world, rank, q, pos)
                dst[h][i] = xv[q, pos]

    def rows_peer(self, rank, world, z, x_peers):
        self.rows(rank, world, z)  # checks the rows arrived, tags the product rows
        R = E // world
        zv = z.view(2, R, MU0, EW)
        dst = [self.by_ptr[p].view(-1, EW) for p in x_peers.tolist()]
        for jr in range(R):
            for pos in range(MU0):
                h, i = peer_index(2, world, rank, jr, pos)
                dst[h][i] = zv[0, jr, pos]

    def decode_partial_ptr(self, rank, world, x, s_ptr):
        # s_ptr: rank 0's gather buffer + this rank's slot
        base = max(p for p in self.by_ptr if p <= s_ptr)
        g = self.by_ptr[base]
        n = (E + 1) * SEG
        off = (s_ptr - base) // 8
        self.decode_partial(rank, world, x, g[off:off + n])


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_virtual_ranks_fused_exchange_places_every_element(world):
    from paper_1503_04955_b200.fourstep import run_virtual_peer

    st = TagPeerStages()
    ranks = [FourStepRank(st, r, world, M, MM, torch.device("cpu"), 4) for r in range(world)]
    st.register(ranks)
    for fs in ranks:  # nothing may be read before the peers wrote it
        fs.z.fill_(-1)
        fs.x.fill_(-1)
    a = torch.zeros(4, dtype=torch.int32)
    out = run_virtual_peer(ranks, a, a)
    assert out.tolist() == [1, 1, 1, 1]
    assert st.calls.count("rows") == world and st.calls.count("columns_inv") == world
    assert st.calls[-1] == "decode"
