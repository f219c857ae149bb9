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
three polynomial exchanges per multiply, plus the final gather.  The exchange is NCCL
all-to-all through torch.distributed (NVLink/NVSwitch on a B200 node).

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


class FourStepRank:
    """Buffers and phases of one rank (all limb buffers are int32 tensors on `device`)."""

    def __init__(self, stages, rank: int, world: int, M: int, m: int, device, product_limbs: int,
                 distributed_decode: bool | None = None):
        lay = stages.layout(world)
        self.stages, self.rank, self.world = stages, rank, world
        self.E = 2 * m
        self.C, self.R, self.ew, self.bw = lay["cols"], lay["rows"], lay["elem_words"], lay["block_words"]
        self.mu0 = 2 * M // self.E
        seg = lay.get("decode_seg", 0)
        self.dist_decode = bool(seg) if distributed_decode is None else (distributed_decode and bool(seg))
        kw = dict(dtype=torch.int32, device=device)
        self.x = torch.empty(2 * self.bw, **kw)  # [2][E][C] columns (phase A/C)
        self.y = torch.empty(2 * self.bw, **kw)  # exchange staging
        self.z = torch.empty(2 * self.bw, **kw)  # [2][R][mu0] rows (phase B)
        if self.dist_decode:
            n_part = (self.E + 1) * seg  # 64-bit window sums of this rank's runs
            self.part = torch.empty(n_part, dtype=torch.int64, device=device)
            self.gath = torch.empty(world * n_part if rank == 0 else 1, dtype=torch.int64, device=device)
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


def make_rank(plan, rank: int, world: int, device=None, distributed_decode: bool | None = None) -> FourStepRank:
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    dp = device_plan(plan, device.index or 0)
    return FourStepRank(DeviceStages(dp), rank, world, plan.M, plan.m, device, dp.info["product_limbs"],
                        distributed_decode)


def _operands(plan, a: int, b: int, device):
    dp = device_plan(plan, device.index or 0)
    nl = dp.info["operand_limbs"]
    A = torch.from_numpy(int_to_u32(int(a), nl).view("int32")).to(device)
    B = torch.from_numpy(int_to_u32(int(b), nl).view("int32")).to(device)
    return A, B


def _to_int(prod: torch.Tensor) -> int:
    return int.from_bytes(prod.cpu().numpy().view("uint32").tobytes(), "little")


def dmul_fourstep(a: int, b: int, group=None) -> int | None:
    """a*b with the multiply split over the ranks of `group` (one GPU per rank, NCCL).

    Every rank passes the same operands; rank 0 returns the product, others None.
    """
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    plan = _plan_and_limbs(a, b)
    dev = torch.device("cuda", torch.cuda.current_device())
    fs = make_rank(plan, rank, world, dev)
    A, B = _operands(plan, a, b, dev)
    prod = run_rank(fs, DistExchange(group), A, B)
    return _to_int(prod) if rank == 0 else None


def dmul_fourstep_virtual(a: int, b: int, world: int, device=None, distributed_decode: bool | None = None) -> int:
    """a*b through the four-step split with `world` ranks emulated on one GPU (tests)."""
    plan = _plan_and_limbs(a, b)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    ranks = [make_rank(plan, r, world, dev, distributed_decode) for r in range(world)]
    A, B = _operands(plan, a, b, dev)
    return _to_int(run_virtual(ranks, A, B))
