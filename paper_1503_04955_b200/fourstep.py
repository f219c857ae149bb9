"""Four-step (Bailey) split of ONE DKSS multiply over G GPUs.

The reference's transform is itself a radix split (bigmul/dkss.py:465-495): with
E = 2m and mu0 = 2M/E, the length-2M vector is an E x mu0 matrix A[j][l] = v[j*mu0 + l];
level 0 transforms the mu0 columns (length-E DFT + twiddle rho^(vv*l), :471-492) and
every deeper level and the base case act inside one of the E rows (:493-495).  So:

  phase A  rank r owns columns [r*C, (r+1)*C), C = mu0/G: encode + level 0 of a and b
           (libdkss dkss_fs_columns_fwd), stored [2][E][C] elements;
  exchange all-to-all: rank r sends rows [h*R, (h+1)*R) of its block to rank h, R = E/G;
           the receiver re-lays [G][R][C] -> [R][mu0] (dkss_block_transpose);
  phase B  rank h owns rows: deeper forward levels of a and b, pointwise r_mul
           (bigmul/dkss.py:544-545) and deeper inverse levels of the product, all local
           (dkss_fs_rows);
  exchange the transpose back (one polynomial);
  phase C  last inverse level on the own columns with the 1/2M scale (dkss_fs_columns_inv);
  decode   distributed (u = 32): every rank turns its columns into the per-limb window sums of
           its logical runs (dkss_fs_decode_partial, 8 bytes per output limb it touches), rank 0
           gathers them, adds the overlapping run ends and resolves the carries
           (dkss_fs_decode_finish); otherwise the product columns are gathered to rank 0,
           re-laid to [E][mu0] and decoded there (dkss_decode_device).

Each rank moves P*(G-1)/G^2 bytes per polynomial per exchange (P = one polynomial),
three polynomial exchanges per multiply, plus the final gather.  Two exchange engines:

  * "peer" (default on GPUs): the exchange is fused into the stores of the phase that
    produces the data -- the first-level pass writes every output element straight into the
    row owner's [2][R][mu0] buffer, the last row-phase pass writes the product rows straight
    into the column owners' [E][C] buffers, and the window sums land in rank 0's gather buffer
    (dkss_fs_columns_fwd_peer / dkss_fs_rows_peer: peer base pointers of the other GPUs'
    buffers, mapped with CUDA IPC, over NVLink).  The transfer overlaps the compute tile by
    tile; no all-to-all, no re-layout kernels, no staging buffer.  Phases are ordered by a
    stream-ordered barrier (a one-element NCCL all-reduce);
  * "alltoall": all-to-all through torch.distributed (NCCL on GPUs) plus dkss_block_transpose
    re-layouts (the baseline the fused path replaces; also the gloo path of the CPU tests).

The orchestration is written against two small interfaces so the same code runs
  * on GPUs with libdkss (``DeviceStages``) and NCCL (``DistExchange``),
  * on one GPU with G emulated ranks (``run_virtual``; the exchange is a local copy), and
  * on CPU under gloo with a stand-in stage object (tests/test_fourstep.py), which checks
    every element lands where the layout says.
"""

from __future__ import annotations

import torch

from .dkss import _plan_for, _MIN_PLAN_BITS, device_plan
from .words import int_to_u32, word_bits


class DeviceStages:
    """The libdkss four-step entry points on torch tensors (int32 views of u32 limbs)."""

    def __init__(self, dp):
        self.dp = dp

    @staticmethod
    def _s() -> int:
        return torch.cuda.current_stream().cuda_stream

    def layout(self, world: int) -> dict:
        return self.dp.fs_layout(world)

    def columns_fwd(self, rank, world, a, b, x):
        self.dp.fs_columns_fwd(rank, world, a.data_ptr(), b.data_ptr(), a.numel(), x.data_ptr(), self._s())

    def rows(self, rank, world, z):
        self.dp.fs_rows(world, z.data_ptr(), self._s())

    def columns_inv(self, rank, world, x):
        self.dp.fs_columns_inv(rank, world, x.data_ptr(), self._s())

    def block_transpose(self, src, dst, n, A, B, run_words):
        self.dp.block_transpose(src.data_ptr(), dst.data_ptr(), n, A, B, run_words, self._s())

    def decode(self, v, out):
        self.dp.decode_device(v.data_ptr(), out.data_ptr(), out.numel(), self._s())

    def decode_partial(self, rank, world, x, s_out):
        self.dp.fs_decode_partial(rank, world, x.data_ptr(), s_out.data_ptr(), self._s())

    def decode_finish(self, world, parts, out):
        self.dp.fs_decode_finish(world, parts.data_ptr(), out.data_ptr(), out.numel(), self._s())

    def columns_fwd_peer(self, rank, world, a, b, x, z_peers):
        self.dp.fs_columns_fwd_peer(rank, world, a.data_ptr(), b.data_ptr(), a.numel(), x.data_ptr(), z_peers.data_ptr(),
                                    self._s())

    def rows_peer(self, rank, world, z, x_peers):
        self.dp.fs_rows_peer(rank, world, z.data_ptr(), x_peers.data_ptr(), self._s())

    def decode_partial_ptr(self, rank, world, x, s_ptr: int):
        self.dp.fs_decode_partial(rank, world, x.data_ptr(), s_ptr, self._s())


class DistExchange:
    """all-to-all / gather over a torch.distributed process group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        # gloo has no all-to-all / gather on CUDA tensors: stage through host memory (tests on a
        # one-GPU box; NCCL takes device tensors directly)
        self.host = dist.get_backend(group) == "gloo"

    def all_to_all(self, out, inp):
        if self.host and out.is_cuda:
            o = torch.empty_like(out, device="cpu")
            self.dist.all_to_all_single(o, inp.cpu(), group=self.group)
            out.copy_(o)
            return
        self.dist.all_to_all_single(out, inp, group=self.group)

    def gather(self, out, inp, rank):
        # out: [G * n] on rank 0 (ignored elsewhere)
        world = self.dist.get_world_size(self.group)
        if self.host and inp.is_cuda:
            o = torch.empty(out.shape, dtype=out.dtype) if rank == 0 else None
            self.gather(o, inp.cpu(), rank)
            if rank == 0:
                out.copy_(o)
            return
        if rank == 0:
            parts = list(out.view(world, -1).unbind(0))
            self.dist.gather(inp, parts, dst=0, group=self.group)
        else:
            self.dist.gather(inp, None, dst=0, group=self.group)


class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer (an IPC buffer) for torch.as_tensor."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


def ipc_tensor(n: int, dtype, device):
    """int32 / int64 tensor of n elements in a CUDA IPC-shareable allocation (dkss_ipc_alloc);
    the allocation lives as long as the tensor (kept in tensor._ipc)."""
    from ._native import IpcBuffer

    size = torch.tensor([], dtype=dtype).element_size()
    buf = IpcBuffer(device.index or 0, max(1, n) * size)
    t = torch.as_tensor(_CudaArray(buf.ptr, max(1, n), "<i4" if size == 4 else "<i8"), device=device)
    t._ipc = buf
    return t


class FourStepRank:
    """Buffers and phases of one rank (all limb buffers are int32 tensors on `device`).

    alloc(n, dtype) makes the buffers other ranks write into under the fused exchange (z, x, the
    gather buffer): torch.empty by default, ipc_tensor for ranks in other processes."""

    def __init__(self, stages, rank: int, world: int, M: int, m: int, device, product_limbs: int,
                 distributed_decode: bool | None = None, alloc=None):
        lay = stages.layout(world)
        self.stages, self.rank, self.world = stages, rank, world
        self.E = 2 * m
        self.C, self.R, self.ew, self.bw = lay["cols"], lay["rows"], lay["elem_words"], lay["block_words"]
        self.mu0 = 2 * M // self.E
        seg = lay.get("decode_seg", 0)
        self.dist_decode = bool(seg) if distributed_decode is None else (distributed_decode and bool(seg))
        kw = dict(dtype=torch.int32, device=device)
        alloc = alloc or (lambda n, dtype: torch.empty(n, dtype=dtype, device=device))
        self.x = alloc(2 * self.bw, torch.int32)  # [2][E][C] columns (phase A/C)
        self.y = torch.empty(2 * self.bw, **kw)  # exchange staging
        self.z = alloc(2 * self.bw, torch.int32)  # [2][R][mu0] rows (phase B)
        if self.dist_decode:
            n_part = (self.E + 1) * seg  # 64-bit window sums of this rank's runs
            self.n_part = n_part
            self.part = torch.empty(n_part, dtype=torch.int64, device=device)
            self.gath = alloc(world * n_part if rank == 0 else 1, torch.int64)
            self.full = None
        else:
            self.full = torch.empty(world * self.bw if rank == 0 else 1, **kw)
            self.gath = torch.empty(world * self.bw if rank == 0 else 1, **kw)
        self.prod = torch.empty(product_limbs if rank == 0 else 1, **kw)

    # one polynomial's share split by destination rank (rows [h*R, (h+1)*R) x C columns)
    def _poly(self, buf, q):
        return buf[q * self.bw:(q + 1) * self.bw]

    def phase_columns(self, a, b):
        self.stages.columns_fwd(self.rank, self.world, a, b, self.x)
        return [self._poly(self.x, 0), self._poly(self.x, 1)], [self._poly(self.y, 0), self._poly(self.y, 1)]

    def phase_rows(self):
        # y[q] = [G src][R][C] -> z[q] = [R][G][C] = [R][mu0]
        self.stages.block_transpose(self.y, self.z, 2, self.world, self.R, self.C * self.ew)
        self.stages.rows(self.rank, self.world, self.z)
        # product rows z[0] = [R][G][C] -> y[0] = [G dst][R][C]
        self.stages.block_transpose(self._poly(self.z, 0), self._poly(self.y, 0), 1, self.R, self.world,
                                    self.C * self.ew)
        return [self._poly(self.y, 0)], [self._poly(self.x, 0)]

    def phase_finish(self):
        """Last inverse level of the own columns (x[0] = [G src][R][C] = [E][C]); returns what
        this rank sends to rank 0: its run window sums (distributed decode) or its columns."""
        self.stages.columns_inv(self.rank, self.world, self._poly(self.x, 0))
        if self.dist_decode:
            self.stages.decode_partial(self.rank, self.world, self._poly(self.x, 0), self.part)
            return self.part
        return self._poly(self.x, 0)

    # fused exchange (peer stores): z_peers / x_peers are device int64 tables of every rank's z / x
    # base address, gath_ptr rank 0's gather buffer as seen from this rank
    def phase_columns_peer(self, a, b, z_peers):
        self.stages.columns_fwd_peer(self.rank, self.world, a, b, self.x, z_peers)

    def phase_rows_peer(self, x_peers):
        self.stages.rows_peer(self.rank, self.world, self.z, x_peers)

    def phase_finish_peer(self, gath_ptr: int):
        self.stages.columns_inv(self.rank, self.world, self._poly(self.x, 0))
        self.stages.decode_partial_ptr(self.rank, self.world, self._poly(self.x, 0),
                                       gath_ptr + 8 * self.rank * self.n_part)

    def decode(self):
        if self.dist_decode:
            # rank 0: gath = [G][E+1][seg] window sums -> product limbs
            self.stages.decode_finish(self.world, self.gath, self.prod)
            return self.prod
        # rank 0: gath = [G][E][C] -> full = [E][G][C] = [E][mu0], then decode
        self.stages.block_transpose(self.gath, self.full, 1, self.world, self.E, self.C * self.ew)
        self.stages.decode(self.full, self.prod)
        return self.prod


def run_rank(fs: FourStepRank, exch, a, b):
    """The whole split multiply on one rank of a real process group; rank 0 returns the
    product limbs (int32 tensor), other ranks None."""
    sends, recvs = fs.phase_columns(a, b)
    for s, r in zip(sends, recvs):
        exch.all_to_all(r, s)
    sends, recvs = fs.phase_rows()
    for s, r in zip(sends, recvs):
        exch.all_to_all(r, s)
    mine = fs.phase_finish()
    exch.gather(fs.gath, mine, fs.rank)
    return fs.decode() if fs.rank == 0 else None


def peer_capable(fs: FourStepRank) -> bool:
    """The fused exchange needs the distributed decode (u = 32) and a row phase of >= 2 levels."""
    return fs.dist_decode and fs.stages.dp.info["levels"] >= 2


class PeerExchange:
    """The fused exchange of one rank in a process group: every rank's z and x (and rank 0's
    gather buffer) are CUDA IPC allocations (FourStepRank(alloc=ipc_tensor)); their handles are
    all-gathered once and mapped here, so the phase kernels store straight into the owners'
    buffers.  barrier() orders the phases across ranks: a one-element all-reduce on the current
    stream under NCCL (no host synchronisation), a host barrier under gloo."""

    def __init__(self, fs: FourStepRank, group=None):
        import torch.distributed as dist

        from ._native import IpcMapping

        self.dist, self.group = dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        dev = fs.z.device
        self.nccl = dist.get_backend(group) == "nccl"
        mine = (fs.z._ipc.handle, fs.x._ipc.handle, fs.gath._ipc.handle if self.rank == 0 else None)
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        self.maps = []  # keep the mappings open

        def addr(r, k, local):
            if r == self.rank:
                return local.data_ptr()
            mp = IpcMapping(dev.index or 0, allh[r][k])
            self.maps.append(mp)
            return mp.ptr

        z = [addr(r, 0, fs.z) for r in range(self.world)]
        x = [addr(r, 1, fs.x) for r in range(self.world)]
        self.z_peers = torch.tensor(z, dtype=torch.int64, device=dev)
        self.x_peers = torch.tensor(x, dtype=torch.int64, device=dev)
        self.gath_ptr = addr(0, 2, fs.gath)
        self._tok = torch.zeros(1, dtype=torch.float32, device=dev if self.nccl else "cpu")

    def barrier(self):
        if self.nccl:
            self.dist.all_reduce(self._tok, group=self.group)
        else:
            torch.cuda.synchronize()
            self.dist.barrier(group=self.group)


def run_rank_peer(fs: FourStepRank, px: PeerExchange, a, b):
    """The split multiply with the exchange fused into the phase kernels' stores (one rank of a
    process group); rank 0 returns the product limbs, other ranks None."""
    fs.phase_columns_peer(a, b, px.z_peers)
    px.barrier()
    fs.phase_rows_peer(px.x_peers)
    px.barrier()
    fs.phase_finish_peer(px.gath_ptr)
    px.barrier()
    return fs.decode() if fs.rank == 0 else None


def run_virtual_peer(ranks, a, b):
    """All G ranks emulated in one process with the fused exchange: the peer tables hold the
    other emulated ranks' buffers (same device), phases run rank after rank."""
    dev = ranks[0].z.device
    z_peers = torch.tensor([fs.z.data_ptr() for fs in ranks], dtype=torch.int64, device=dev)
    x_peers = torch.tensor([fs.x.data_ptr() for fs in ranks], dtype=torch.int64, device=dev)
    for fs in ranks:
        fs.phase_columns_peer(a, b, z_peers)
    for fs in ranks:
        fs.phase_rows_peer(x_peers)
    g = ranks[0].gath.data_ptr()
    for fs in ranks:
        fs.phase_finish_peer(g)
    return ranks[0].decode()


def _local_all_to_all(outs, ins):
    """ins[r] / outs[h]: per-rank buffers of G equal chunks; outs[h][r] = ins[r][h]."""
    G = len(ins)
    for h in range(G):
        o = outs[h].view(G, -1)
        for r in range(G):
            o[r].copy_(ins[r].view(G, -1)[h])


def run_virtual(ranks, a, b):
    """All G ranks emulated in one process (one device): same phases, exchange by copies."""
    G = len(ranks)
    steps = [fs.phase_columns(a, b) for fs in ranks]
    for q in range(len(steps[0][0])):
        _local_all_to_all([s[1][q] for s in steps], [s[0][q] for s in steps])
    steps = [fs.phase_rows() for fs in ranks]
    for q in range(len(steps[0][0])):
        _local_all_to_all([s[1][q] for s in steps], [s[0][q] for s in steps])
    mine = [fs.phase_finish() for fs in ranks]
    g = ranks[0].gath.view(G, -1)
    for r in range(G):
        g[r].copy_(mine[r])
    return ranks[0].decode()


# ---------------------------------------------------------------------------
# public entry points

def _plan_and_limbs(a: int, b: int):
    n_bits = max(int(a).bit_length(), int(b).bit_length(), _MIN_PLAN_BITS)
    plan = _plan_for(n_bits, word_bits())
    return plan


def make_rank(plan, rank: int, world: int, device=None, distributed_decode: bool | None = None,
              ipc: bool = False) -> FourStepRank:
    """ipc=True: the buffers other ranks write into are CUDA IPC allocations (PeerExchange)."""
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    dp = device_plan(plan, device.index or 0)
    alloc = (lambda n, dtype: ipc_tensor(n, dtype, device)) if ipc else None
    return FourStepRank(DeviceStages(dp), rank, world, plan.M, plan.m, device, dp.info["product_limbs"],
                        distributed_decode, alloc=alloc)


def _operands(plan, a: int, b: int, device):
    dp = device_plan(plan, device.index or 0)
    nl = dp.info["operand_limbs"]
    A = torch.from_numpy(int_to_u32(int(a), nl).view("int32")).to(device)
    B = torch.from_numpy(int_to_u32(int(b), nl).view("int32")).to(device)
    return A, B


def _to_int(prod: torch.Tensor) -> int:
    return int.from_bytes(prod.cpu().numpy().view("uint32").tobytes(), "little")


def dmul_fourstep(a: int, b: int, group=None, exchange: str = "peer") -> int | None:
    """a*b with the multiply split over the ranks of `group` (one GPU per rank).

    exchange "peer": fused into the phase kernels' stores over CUDA IPC peer memory (falls back to
    "alltoall" for plans it does not cover: u != 32 or a single transform level); "alltoall":
    all-to-all through torch.distributed.  Every rank passes the same operands; rank 0 returns the product,
    others None."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    plan = _plan_and_limbs(a, b)
    dev = torch.device("cuda", torch.cuda.current_device())
    fs = make_rank(plan, rank, world, dev, ipc=exchange == "peer")
    A, B = _operands(plan, a, b, dev)
    if exchange == "peer" and peer_capable(fs):
        prod = run_rank_peer(fs, PeerExchange(fs, group), A, B)
    else:
        prod = run_rank(fs, DistExchange(group), A, B)
    return _to_int(prod) if rank == 0 else None


def dmul_fourstep_virtual(a: int, b: int, world: int, device=None, distributed_decode: bool | None = None,
                          exchange: str = "copy") -> int:
    """a*b through the four-step split with `world` ranks emulated on one GPU (tests):
    exchange "copy" (all-to-all by local copies + re-layout kernels) or "peer" (fused stores)."""
    plan = _plan_and_limbs(a, b)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    ranks = [make_rank(plan, r, world, dev, distributed_decode) for r in range(world)]
    A, B = _operands(plan, a, b, dev)
    if exchange == "peer":
        if not peer_capable(ranks[0]):
            raise ValueError("the fused exchange needs u = 32 and >= 2 transform levels")
        return _to_int(run_virtual_peer(ranks, A, B))
    return _to_int(run_virtual(ranks, A, B))
