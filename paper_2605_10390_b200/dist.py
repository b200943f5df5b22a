"""Multi-GPU keys-only u16 sort: one process per GPU, torch.distributed for the
plumbing (NCCL over NVLink on B200), the local steps in libfractalsort.so.

SURVEY.md §8(e).  Every rank holds a shard (a contiguous slice of the input by
global index).  Per-shard histograms form a sum monoid, so ONE collective merges
them exactly — the Global Histogram Update of PAPER.md:91-92 taken across GPUs —
and the exact output partition needs no sampling: rank d owns global sorted
positions [floor(d*N/G), floor((d+1)*N/G)) (ledger 23).

mode "B" (compressed exchange, the scaling path): the exchanged form of a shard
    is its 512 KiB histogram.  all_reduce(hist) -> scan -> expand the rank's own
    output range.  NVLink carries 512 KiB per rank, HBM 4 B/key of the rank's
    share: near-linear by construction.
mode "A" (payload exchange by key range, the literal c4 reading): local sort of
    the shard, all_gather of the histograms, exact send counts (fs_send_counts:
    lower rank first for equal keys), all_to_all_single of the key
    bytes, and a local sort of what arrived.
mode "P" (fused expand-to-peer): all_gather of the
    histograms, then every rank writes each of its own keys straight to its
    final sorted position in the owning rank's output buffer, mapped into its
    address space with CUDA IPC (NVLink / NVSwitch peer stores,
    fs_expand_to_peers_u16); a barrier ends the exchange.  The payload crosses
    NVLink once and no rank sorts anything.

``ops`` supplies the local steps.  The default, CudaOps, calls the library's
kernels through the binding; the gloo tests on CPU inject their own stand-ins
(from tests/), which exercises exactly this module's orchestration.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class CudaOps:
    """Local steps on the current CUDA device (libfractalsort.so)."""

    def histogram_u16(self, keys):
        from . import histogram_u16
        return histogram_u16(keys)                  # int64[65536]

    def exclusive_scan(self, hist):
        from . import exclusive_scan
        return exclusive_scan(hist)                 # int64[65537]

    def expand_u16(self, prefix, begin, end):
        from . import expand_u16
        return expand_u16(prefix, begin, end)

    def sort_keys(self, keys):
        from . import sort_keys
        return sort_keys(keys)

    def send_counts(self, hist_all, g):
        from . import send_counts
        return send_counts(hist_all, g)             # int64[G]

    def expand_to_peers(self, hist_all, g, dest):
        from . import expand_to_peers_u16
        expand_to_peers_u16(hist_all, g, dest)

    def synchronize(self, device):
        torch.cuda.synchronize(device)


class PeerBuffers:
    """Every rank's output buffer, mapped into every rank (CUDA IPC through
    torch's tensor sharing; peer access over NVLink is enabled by the mapping).
    Buffers hold ceil(N / G) keys (every rank's range fits) and are reallocated,
    collectively, only when a larger N arrives."""

    def __init__(self, device, group=None):
        self.device, self.group, self.capacity, self.views = device, group, 0, None

    def buffers(self, per_rank: int):
        if per_rank > self.capacity:
            from torch.multiprocessing.reductions import reduce_tensor
            world, rank = dist.get_world_size(self.group), dist.get_rank(self.group)
            own = torch.empty(max(per_rank, 1), dtype=torch.uint16, device=self.device)
            handles = [None] * world
            dist.all_gather_object(handles, reduce_tensor(own) if world > 1 else None, group=self.group)
            self.views = [own if r == rank else handles[r][0](*handles[r][1]) for r in range(world)]
            self.capacity = per_rank
        return self.views


def output_range(rank: int, world: int, n_total: int):
    """Rank's global sorted positions [floor(r N / G), floor((r+1) N / G))."""
    return (n_total * rank) // world, (n_total * (rank + 1)) // world


def _total_keys(n_local: int, device, group) -> int:
    t = torch.tensor([n_local], dtype=torch.int64, device=device)
    dist.all_reduce(t, group=group)
    return int(t.item())


def sort_keys_u16(shard: torch.Tensor, group=None, mode: str = "B", ops=None, peers=None):
    """Sort the union of all ranks' shards; returns (this rank's slice of the sorted
    output, (begin, end) global positions of that slice).  mode "P" writes into
    ``peers.buffers(...)`` (a PeerBuffers by default; pass one to reuse the
    mappings across calls) and returns a view of this rank's buffer."""
    if shard.dtype != torch.uint16 or shard.dim() != 1:
        raise TypeError("shard must be a 1-D uint16 tensor")
    ops = ops or CudaOps()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = shard.device
    if mode == "B":
        hist = ops.histogram_u16(shard)
        dist.all_reduce(hist, group=group)
        prefix = ops.exclusive_scan(hist)
        n_total = int(prefix[-1].item())
        begin, end = output_range(rank, world, n_total)
        return ops.expand_u16(prefix, begin, end), (begin, end)
    if mode == "A":
        hist = ops.histogram_u16(shard)
        gathered = [torch.empty_like(hist) for _ in range(world)]
        dist.all_gather(gathered, hist, group=group)
        hist_all = torch.stack(gathered)                       # G x 65536
        n_total = int(hist_all.sum().item())
        begin, end = output_range(rank, world, n_total)
        send = ops.send_counts(hist_all, rank)                 # keys of this rank per destination
        send_list = [int(x) for x in send.tolist()]
        recv = torch.empty(world, dtype=torch.int64, device=dev)
        dist.all_to_all_single(recv, send.to(torch.int64), group=group)
        recv_list = [int(x) for x in recv.tolist()]
        assert sum(recv_list) == end - begin
        local_sorted = ops.sort_keys(shard) if shard.numel() else shard
        recv_buf = torch.empty(end - begin, dtype=torch.uint16, device=dev)
        # NCCL/gloo have no 16-bit integer type: exchange bytes.
        dist.all_to_all_single(recv_buf.view(torch.uint8), local_sorted.view(torch.uint8),
                               output_split_sizes=[2 * c for c in recv_list],
                               input_split_sizes=[2 * c for c in send_list], group=group)
        out = ops.sort_keys(recv_buf) if recv_buf.numel() else recv_buf
        return out, (begin, end)
    if mode == "P":
        hist = ops.histogram_u16(shard)
        gathered = [torch.empty_like(hist) for _ in range(world)]
        dist.all_gather(gathered, hist, group=group)
        hist_all = torch.stack(gathered)                       # G x 65536
        n_total = int(hist_all.sum().item())
        begin, end = output_range(rank, world, n_total)
        if peers is None:
            peers = PeerBuffers(dev, group)
        dest = peers.buffers(-(-n_total // world))
        ops.expand_to_peers(hist_all, rank, dest)
        ops.synchronize(dev)
        dist.barrier(group=group)                              # every producer has finished writing
        return dest[rank][:end - begin], (begin, end)
    raise ValueError(f"unknown mode {mode!r}")
