"""Multi-GPU keys-only u16 sort: one process per GPU, torch.distributed for the
plumbing (NCCL over NVLink on B200), the local steps in libfractalsort.so.

SURVEY.md §8(e).  Every rank holds a shard (a contiguous slice of the input by
global index).  Per-shard histograms form a sum monoid, so ONE collective merges
them exactly — the Global Histogram Update of PAPER.md:91-92 taken across GPUs —
and the exact output partition needs no sampling: rank d owns global sorted
positions [floor(d*N/G), floor((d+1)*N/G)) (ledger 23).

mode "B" (compressed exchange, the scaling path): the exchanged form of a shard
    is its histogram, as the sort's two-level prefix (slice-local prefixes +
    slice totals, linear in the counts).  all_reduce of those 65,664 counters
    -> expand the rank's own output range (no scan kernel: the slice bases are
    folded into the expansion).  NVLink carries 513 KiB per rank, HBM 4 B/key of
    the rank's share: near-linear by construction.
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

mode "N" (NVLS): mode B with the all_reduce done by the
    NVSwitch.  Each rank's histogram kernel writes its two-level prefix straight
    into its own GPU memory bound into one multicast object (MulticastBuffer);
    fs_allreduce_multicast_u64 then reads the sum over ranks through the
    multicast address (multimem.ld_reduce: the switch adds the G copies) after a
    barrier carried by the same kernel (multimem.red on a flag word).  No NCCL
    kernel, no staging copy; 513 KiB per rank read through the switch.

``ops`` supplies the local steps.  The default, CudaOps, calls the library's
kernels through the binding; the gloo tests on CPU inject their own stand-ins
(from tests/), which exercises exactly this module's orchestration.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


class CudaOps:
    """Local steps on the current CUDA device (libfractalsort.so)."""

    def histogram_u16(self, keys):
        from . import histogram_u16
        return histogram_u16(keys)                  # int64[65536]

    def histogram_prefix_u16(self, keys):
        from . import histogram_prefix_u16
        return histogram_prefix_u16(keys)           # int64[65536 + 128]

    def expand_prefix_u16(self, prefix2, begin, end):
        from . import expand_prefix_u16
        return expand_prefix_u16(prefix2, begin, end)

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

    def sort_pairs(self, keys, vals):
        from . import sort_pairs
        return sort_pairs(keys, vals)

    def bound_u64(self, sorted_keys, queries, upper):
        from . import bound_u64
        return bound_u64(sorted_keys, queries, upper)            # int64 counts

    def expand_to_peers(self, hist_all, g, dest):
        from . import expand_to_peers_u16
        expand_to_peers_u16(hist_all, g, dest)

    def histogram16_u64(self, keys, shift, width):
        from . import histogram16_u64
        return histogram16_u64(keys, shift, width)      # int64[2^width]

    def select_bins_u64(self, keys, shift, width, bins, cap):
        from . import select_bins_u64
        return select_bins_u64(keys, shift, width, bins, cap)

    def sort_keys_u64(self, keys):
        from . import sort_keys
        return sort_keys(keys)

    def digit_counts_sorted_u64(self, sorted_keys, prefixes, shift, width):
        from . import digit_counts_sorted_u64
        return digit_counts_sorted_u64(sorted_keys, prefixes, shift, width)   # int64[len, 2^width]

    def pair_exchange(self, keys, vals, splitters, G):
        from . import PairExchange
        return PairExchange(keys, vals, splitters, G)

    def histogram_prefix_u16_to(self, keys, out_ptr):
        from . import histogram_prefix_u16
        histogram_prefix_u16(keys, out_ptr=out_ptr)

    def allreduce_multicast(self, src_mc, dst, flag_mc, flag_local, target):
        from . import allreduce_multicast_u64
        return allreduce_multicast_u64(src_mc, dst, flag_mc, flag_local, target)   # (dst, timed_out flag)

    def synchronize(self, device):
        torch.cuda.synchronize(device)


class PeerBuffers:
    """Every rank's output buffer, mapped into every rank (CUDA IPC through
    torch's tensor sharing; peer access over NVLink is enabled by the mapping).
    Buffers hold ceil(N / G) elements (every rank's range fits) and are
    reallocated, collectively, only when a larger N arrives.  dtype: uint16
    keys (mode "P"), uint64 keys / uint32 values (pairs, mode "P")."""

    _STORAGE = {torch.uint16: torch.int16, torch.uint32: torch.int32, torch.uint64: torch.int64}

    def __init__(self, device, group=None, dtype=torch.uint16):
        self.device, self.group, self.dtype, self.capacity, self.views = device, group, dtype, 0, None

    def buffers(self, per_rank: int):
        if per_rank > self.capacity:
            from torch.multiprocessing.reductions import reduce_tensor
            world, rank = dist.get_world_size(self.group), dist.get_rank(self.group)
            own = torch.empty(max(per_rank, 1), dtype=self._STORAGE[self.dtype], device=self.device)
            handles = [None] * world
            dist.all_gather_object(handles, reduce_tensor(own) if world > 1 else None, group=self.group)
            views = [own if r == rank else handles[r][0](*handles[r][1]) for r in range(world)]
            self.views = [v.view(self.dtype) for v in views]
            self.capacity = per_rank
        return self.views


def share_fd(fd, group=None):
    """Rank 0's file descriptor ``fd``, duplicated into every rank of ``group``
    (SCM_RIGHTS over an abstract Unix socket; the socket name travels through
    the process group).  Returns the local descriptor (rank 0: ``fd`` itself).
    Used for the multicast object's POSIX handle (MulticastBuffer)."""
    import socket
    import uuid
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if world == 1:
        return fd
    name = [None]
    srv = None
    if rank == 0:
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        addr = "\0fractalsort-fd-" + uuid.uuid4().hex
        srv.bind(addr)
        srv.listen(world)
        srv.settimeout(120)                                # a peer that never connects raises here, not a hang
        name = [addr]
    dist.broadcast_object_list(name, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    if rank == 0:
        try:
            for _ in range(world - 1):
                conn, _ = srv.accept()
                with conn:
                    socket.send_fds(conn, [b"f"], [fd])
                    conn.recv(1)                                   # the peer holds its copy
        finally:
            srv.close()
        return fd
    with socket.socket(socket.AF_UNIX, socket.SOCK_STREAM) as c:
        c.settimeout(120)
        c.connect(name[0])
        _, fds, _, _ = socket.recv_fds(c, 1, 1)
        c.sendall(b"k")
    if len(fds) != 1:
        raise RuntimeError(f"share_fd: rank {rank} received {len(fds)} descriptors")
    return fds[0]


def multicast_step(calls: int, world: int, uc: int, mc: int, half_bytes: int, flag_off: int):
    """Call number ``calls`` (1, 2, ...) of fs_allreduce_multicast_u64 on a
    MulticastBuffer: (local half, multicast half, flag multicast, flag local,
    target).  Halves alternate by call parity, so a rank rewrites a half only two
    calls after it was read (every rank has arrived at the call in between);
    target = G x calls, the flag's value once every rank has arrived (mod 2^32:
    the kernel compares wrap-safely)."""
    h = calls & 1
    return (uc + h * half_bytes, mc + h * half_bytes, mc + flag_off, uc + flag_off, (world * calls) & 0xFFFFFFFF)


class MulticastBuffer:
    """``count`` u64 per half, two halves (alternated by call parity), and a u32
    flag, in every rank's GPU memory, all bound at the same offsets into ONE
    NVSwitch multicast object (driver API through cuda-python: cuMulticastCreate
    on rank 0, POSIX-fd export shared with share_fd, cuMulticastAddDevice on
    every rank, a barrier, cuMemCreate + cuMulticastBindMem, then unicast and
    multicast virtual mappings).  ``step()`` returns the addresses of the next
    call of fs_allreduce_multicast_u64: (local half pointer, multicast half
    pointer, flag multicast pointer, flag local pointer, target)."""

    def __init__(self, count: int, device, group=None):
        from cuda.bindings import driver as cu
        self._cu, self.count, self.group = cu, int(count), group
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.device = torch.device(device)
        self._mem = None
        torch.cuda.set_device(self.device)
        torch.cuda.synchronize(self.device)            # the primary context is current on this thread

        def ok(res, what):
            err = res[0] if isinstance(res, tuple) else res
            if err != cu.CUresult.CUDA_SUCCESS:
                raise RuntimeError(f"MulticastBuffer: {what} failed: {err}")
            return res[1] if isinstance(res, tuple) and len(res) == 2 else res

        def agreed(step):
            """This rank's part of a setup step, then a MIN all-reduce of the success
            flags: if any rank failed, every rank raises here (none is left waiting
            in a later collective).  Doubles as the barrier between steps."""
            err = None
            try:
                step()
            except Exception as e:  # noqa: BLE001 -- re-raised below, after the agreement
                err = e
            if self.world > 1:
                on_dev = dist.get_backend(group) == "nccl"
                flag = torch.tensor([0 if err else 1], dtype=torch.int32, device=self.device if on_dev else "cpu")
                dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
                if err is None and int(flag.item()) == 0:
                    raise RuntimeError("MulticastBuffer: another rank failed a setup step")
            if err is not None:
                raise err

        fdtype = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        self.half_bytes = -(-self.count * 8 // 256) * 256
        self.flag_off = 2 * self.half_bytes
        need = self.flag_off + 256
        st = {}

        def query():
            st["cudev"] = ok(cu.cuDeviceGet(self.device.index), "cuDeviceGet")
            if ok(cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED,
                                          st["cudev"]), "cuDeviceGetAttribute") != 1:
                raise RuntimeError("MulticastBuffer: the device has no multicast (NVLS) support")
            aprop = cu.CUmemAllocationProp()
            aprop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
            aprop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
            aprop.location.id = self.device.index
            aprop.requestedHandleTypes = fdtype
            agran = ok(cu.cuMemGetAllocationGranularity(
                aprop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "granularity")
            mprop = cu.CUmulticastObjectProp()
            mprop.numDevices = self.world
            mprop.handleTypes = fdtype
            mprop.size = need
            mgran = ok(cu.cuMulticastGetGranularity(
                mprop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED), "multicast granularity")
            st["gran"] = max(int(agran), int(mgran))
            self.size = -(-need // st["gran"]) * st["gran"]
            mprop.size = self.size
            st["aprop"], st["mprop"] = aprop, mprop

        def create():
            st["fd"] = None
            if self.rank == 0:
                self._mc = ok(cu.cuMulticastCreate(st["mprop"]), "cuMulticastCreate")
                if self.world > 1:
                    st["fd"] = ok(cu.cuMemExportToShareableHandle(self._mc, fdtype, 0), "export")

        def import_():
            if self.rank != 0:
                self._mc = ok(cu.cuMemImportFromShareableHandle(st["fd_local"], fdtype), "import")
            os.close(st["fd_local"])

        def add_device():
            ok(cu.cuMulticastAddDevice(self._mc, st["cudev"]), "cuMulticastAddDevice")

        def bind_and_map():
            gran = st["gran"]
            self._mem = ok(cu.cuMemCreate(self.size, st["aprop"], 0), "cuMemCreate")
            ok(cu.cuMulticastBindMem(self._mc, 0, self._mem, 0, self.size, 0), "cuMulticastBindMem")
            access = cu.CUmemAccessDesc()
            access.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
            access.location.id = self.device.index
            access.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
            self.uc = int(ok(cu.cuMemAddressReserve(self.size, gran, 0, 0), "reserve (unicast)"))
            ok(cu.cuMemMap(self.uc, self.size, 0, self._mem, 0), "map (unicast)")
            ok(cu.cuMemSetAccess(self.uc, self.size, [access], 1), "access (unicast)")
            self.mc = int(ok(cu.cuMemAddressReserve(self.size, gran, 0, 0), "reserve (multicast)"))
            ok(cu.cuMemMap(self.mc, self.size, 0, self._mc, 0), "map (multicast)")
            ok(cu.cuMemSetAccess(self.mc, self.size, [access], 1), "access (multicast)")
            ok(cu.cuMemsetD8(self.uc, 0, self.size), "zero")
            ok(cu.cuCtxSynchronize(), "synchronize")

        def share():
            st["fd_local"] = share_fd(st["fd"], group)     # its socket steps time out instead of hanging

        agreed(query)
        agreed(create)
        if self.world > 1:
            agreed(share)
            agreed(import_)
        self._cudev = st["cudev"]
        agreed(add_device)        # every device added before any binding
        agreed(bind_and_map)      # every flag zeroed before any arrival
        self.calls = 0

    def step(self):
        """Addresses for the next fs_allreduce_multicast_u64 call (see the class doc)."""
        self.calls += 1
        return multicast_step(self.calls, self.world, self.uc, self.mc, self.half_bytes, self.flag_off)

    def close(self):
        """Unmap and release this rank's memory and handle.  Other ranks read this
        rank's memory through the switch: call it only once every rank's last
        fs_allreduce_multicast_u64 on the buffer has completed (e.g. after a barrier)."""
        cu = self._cu
        if getattr(self, "_mem", None) is None:
            return
        torch.cuda.synchronize(self.device)
        cu.cuMemUnmap(self.mc, self.size)
        cu.cuMemUnmap(self.uc, self.size)
        cu.cuMemAddressFree(self.mc, self.size)
        cu.cuMemAddressFree(self.uc, self.size)
        cu.cuMulticastUnbind(self._mc, self._cudev, 0, self.size)
        cu.cuMemRelease(self._mem)
        cu.cuMemRelease(self._mc)
        self._mem = None


def output_range(rank: int, world: int, n_total: int):
    """Rank's global sorted positions [floor(r N / G), floor((r+1) N / G))."""
    return (n_total * rank) // world, (n_total * (rank + 1)) // world


def _own_range_count(hist_all, rank, begin, end) -> int:
    """How many of rank's keys land in its own output range [begin, end)
    (lower rank first for equal keys: global position P[v] + S_<rank[v] + j)."""
    C = hist_all.to("cpu", torch.int64)
    tot = C.sum(dim=0)
    P = torch.cumsum(tot, 0) - tot                              # exclusive scan
    S = C[:rank].sum(dim=0) if rank else torch.zeros_like(tot)
    lo = P + S                                                  # first global position of rank's keys of v
    hi = lo + C[rank]
    return int((torch.clamp(torch.minimum(hi, torch.full_like(hi, end)) - torch.maximum(lo, torch.full_like(lo, begin)),
                            min=0)).sum().item())


def _total_keys(n_local: int, device, group) -> int:
    t = torch.tensor([n_local], dtype=torch.int64, device=device)
    dist.all_reduce(t, group=group)
    return int(t.item())


def _mark(events, name):
    if events is not None:
        events[name].record()


def sort_keys_u16(shard: torch.Tensor, group=None, mode: str = "B", ops=None, peers=None, events=None, stats=None):
    """Sort the union of all ranks' shards; returns (this rank's slice of the sorted
    output, (begin, end) global positions of that slice).  mode "P" writes into
    ``peers.buffers(...)`` (a PeerBuffers by default; pass one to reuse the
    mappings across calls) and returns a view of this rank's buffer.  mode "N"
    takes ``peers`` as a MulticastBuffer(65,664, device, group) (created on each
    call if None; pass one to reuse it).

    Measurement hooks (bench.py): ``events`` -- a dict with CUDA events "x0" and
    "x1", recorded on the current stream around the payload exchange (modes A and
    P: the all-to-all of the key bytes / the expand-to-peers kernel and the
    barrier after it); ``stats`` -- a dict that receives "sent_bytes", the bytes
    this rank sends to other ranks."""
    if shard.dtype != torch.uint16 or shard.dim() != 1:
        raise TypeError("shard must be a 1-D uint16 tensor")
    ops = ops or CudaOps()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = shard.device
    if mode == "B":
        prefix2 = ops.histogram_prefix_u16(shard)
        dist.all_reduce(prefix2, group=group)
        n_total = int(prefix2[65536:].sum().item())
        begin, end = output_range(rank, world, n_total)
        return ops.expand_prefix_u16(prefix2, begin, end), (begin, end)
    if mode == "N":
        own = peers is None                                    # a buffer made for this call is released after it
        if own:
            peers = MulticastBuffer(65536 + 128, dev, group)
        uc_half, mc_half, flag_mc, flag_local, target = peers.step()
        ops.histogram_prefix_u16_to(shard, uc_half)
        prefix2 = torch.empty(65536 + 128, dtype=torch.int64, device=dev)
        _mark(events, "x0")
        _, timed_out = ops.allreduce_multicast(mc_half, prefix2, flag_mc, flag_local, target)
        _mark(events, "x1")
        n_total = int(prefix2[65536:].sum().item())
        if int(timed_out.item()):   # (a buffer made here is left mapped: a peer may still be reading it)
            raise RuntimeError(f"mode N: rank {rank}: the other ranks did not reach the multicast all-reduce")
        if own:
            if world > 1:
                dist.barrier(group=group)                      # every rank's switch reads of this memory are done
            peers.close()
        begin, end = output_range(rank, world, n_total)
        return ops.expand_prefix_u16(prefix2, begin, end), (begin, end)
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
        if sum(recv_list) != end - begin:
            raise RuntimeError(f"mode A: rank {rank} receives {sum(recv_list)} keys for a range of {end - begin}")
        local_sorted = ops.sort_keys(shard) if shard.numel() else shard
        recv_buf = torch.empty(end - begin, dtype=torch.uint16, device=dev)
        if stats is not None:
            stats["sent_bytes"] = 2 * (sum(send_list) - send_list[rank])
        # NCCL/gloo have no 16-bit integer type: exchange bytes.
        _mark(events, "x0")
        dist.all_to_all_single(recv_buf.view(torch.uint8), local_sorted.view(torch.uint8),
                               output_split_sizes=[2 * c for c in recv_list],
                               input_split_sizes=[2 * c for c in send_list], group=group)
        _mark(events, "x1")
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
        if stats is not None:
            stats["sent_bytes"] = 2 * (int(hist_all[rank].sum().item()) - _own_range_count(hist_all, rank, begin, end))
        _mark(events, "x0")
        ops.expand_to_peers(hist_all, rank, dest)
        _mark(events, "x1")
        ops.synchronize(dev)
        dist.barrier(group=group)                              # every producer has finished writing
        return dest[rank][:end - begin], (begin, end)
    raise ValueError(f"unknown mode {mode!r}")


# ---------------------------------------------------------------- pairs (Mode A)
def _u64_tensor(values, device):
    import numpy as np
    return torch.from_numpy(np.array(values, dtype=np.uint64).view(np.int64)).to(device).view(torch.uint64)


def _levels(key_bits: int):
    """(shift, width) of the digits from the top, 16 bits each (the last one narrower)."""
    out, hi = [], key_bits
    while hi > 0:
        w = min(16, hi)
        out.append((hi - w, w))
        hi -= w
    return out


def splitter_level1(H, bounds, shift):
    """Top digits of the K_d and L_d = #keys below them, from the global level-1 histogram H."""
    import numpy as np
    H = np.asarray(H, dtype=np.int64)
    cum = np.cumsum(H)
    K, L = [], []
    for t in bounds:
        v = int(np.searchsorted(cum, t, side="right"))
        K.append(v << shift)
        L.append(int(cum[v] - H[v]))
    return K, L


def splitter_refine(Hl, bounds, K, L, shift):
    """One more digit of every K_d (in place) from the global histograms Hl[d] of
    that digit among the keys sharing K_d's digits so far."""
    import numpy as np
    Hl = np.asarray(Hl, dtype=np.int64)
    for j in range(len(bounds)):
        cj = np.cumsum(Hl[j])
        v = int(np.searchsorted(cj, bounds[j] - L[j], side="right"))
        L[j] += int(cj[v] - Hl[j][v])
        K[j] |= v << shift


def pair_cuts(T_all, K, L, bounds, nr):
    """Every rank's class-order cuts (G + 1 each) of the fused exchange, from all
    ranks' class totals T_all[r][c] (c = 2d: K_{d-1} < key < K_d; 2d + 1: key ==
    K_d, lowest d): owner d's share starts inside the tie class of K_{d-1}, after
    that class's T = s - L ties below the boundary, lower ranks first."""
    import numpy as np
    T_all = np.asarray(T_all, dtype=np.int64)
    world = len(nr)
    first = [next(i for i in range(world - 1) if K[i] == K[j]) for j in range(world - 1)]
    cuts_all = []
    for r in range(world):
        start = np.concatenate([[0], np.cumsum(T_all[r])])
        cuts = [0]
        for j in range(world - 1):
            c = 2 * first[j] + 1                                    # the tie class of value K_j
            take = min(max(bounds[j] - L[j] - int(T_all[:r, c].sum()), 0), int(T_all[r, c]))
            cuts.append(int(start[c]) + take)
        cuts.append(int(nr[r]))
        cuts_all.append(cuts)
    return cuts_all


def _exact_splitters(ops, level1_local, candidates, N: int, world: int, key_bits: int, group):
    """K_d, L_d for every rank boundary s_d = floor(dN/G), d = 1..G-1: K_d is the key
    of the element at global sorted position s_d and L_d = #keys < K_d over all
    ranks, found digit by digit from compressed histograms (
    no sampling, one all-reduce per 16-bit level -- at most 4 for 64-bit keys).
    level1_local: this rank's int64 histogram of the top digit over all its keys;
    candidates(bins): this rank's keys whose top digit is in bins, ascending."""
    levels = _levels(key_bits)
    bounds = [(N * d) // world for d in range(1, world)]
    h = level1_local.to(torch.int64).clone()
    dist.all_reduce(h, group=group)
    K, L = splitter_level1(h.cpu().numpy(), bounds, levels[0][0])
    if len(levels) > 1:
        cand = candidates(sorted({k >> levels[0][0] for k in K}))
        for shift, width in levels[1:]:
            hl = ops.digit_counts_sorted_u64(cand, K, shift, width).to(torch.int64)
            dist.all_reduce(hl, group=group)
            splitter_refine(hl.cpu().numpy(), bounds, K, L, shift)
    return K, L


def sort_pairs_u64_u32(keys: torch.Tensor, vals: torch.Tensor, group=None, ops=None, key_bits: int = 64,
                       mode: str = "P", peers=None, events=None, stats=None):
    """Stable sort of the (u64 key, u32 value) pairs of all ranks (SURVEY.md §8(e)
    pairs, §8(f) NEXT-2): the ranks' shards are contiguous slices of the input in
    rank order, so the global stable order breaks key ties by (rank, local
    position).  Returns (this rank's slice of the sorted pairs, (begin, end)).

    Exact splitters, no sampling (_exact_splitters): K_d at every rank boundary
    s_d = floor(dN/G) from one all-reduced 16-bit histogram per level; the ties
    at K_d below the boundary, T_d = s_d - L_d, are split by source rank, then
    local order (ledger 13, 23).
    mode "P" (fused exchange, the default): no local sort first -- every pair is
    classified against the splitters (fs_pair_classes_u64: one all_gather of the
    2G - 1 class totals gives every rank's cuts) and stored straight into its
    owner's CUDA-IPC-mapped receive buffer (fs_pair_scatter_u64_u32, peer stores
    over NVLink); each owner then sorts what arrived, once.
    mode "A" (payload all-to-all): stable local sort, cuts from the sorted shard,
    NCCL all_to_all of keys and values, stable local sort of what arrived.
    ``peers``: (keys, values) PeerBuffers to reuse across calls (mode "P").
    ``events`` / ``stats``: as in sort_keys_u16 (around the payload exchange;
    "sent_bytes" = 12 B per pair this rank sends to other ranks).
    """
    import numpy as np
    if keys.dtype != torch.uint64 or vals.dtype != torch.uint32 or keys.numel() != vals.numel():
        raise TypeError("uint64 keys and uint32 values of equal length expected")
    if not 1 <= key_bits <= 64:
        raise ValueError("key_bits must be in 1..64")
    ops = ops or CudaOps()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = keys.device
    n_local = keys.numel()
    sizes = torch.tensor([n_local], dtype=torch.int64, device=dev)
    all_sizes = [torch.empty_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    nr = [int(t.item()) for t in all_sizes]
    N = sum(nr)
    begin, end = output_range(rank, world, N)
    if world == 1:
        return (ops.sort_pairs(keys, vals) if n_local else (keys, vals)), (begin, end)
    shift1, width1 = _levels(key_bits)[0]
    bounds = [(N * d) // world for d in range(1, world)]       # s_d, d = 1 .. G-1
    if mode == "P":
        level1 = ops.histogram16_u64(keys, shift1, width1)

        def candidates(bins):
            cap = int(level1[torch.tensor(bins, dtype=torch.int64, device=level1.device)].sum().item())
            c = ops.select_bins_u64(keys, shift1, width1, bins, cap)
            return ops.sort_keys_u64(c) if c.numel() else c
        K, L = _exact_splitters(ops, level1, candidates, N, world, key_bits, group)
        ex = ops.pair_exchange(keys, vals, K, world)
        tot = torch.tensor(ex.classes(), dtype=torch.int64, device=dev)
        gathered = [torch.empty_like(tot) for _ in range(world)]
        dist.all_gather(gathered, tot, group=group)
        T_all = np.stack([t.cpu().numpy() for t in gathered]).astype(np.int64)   # [rank][class]
        cuts_all = pair_cuts(T_all, K, L, bounds, nr)
        cuts = cuts_all[rank]
        if any(cuts[d] > cuts[d + 1] for d in range(world)):
            raise RuntimeError(f"mode P: rank {rank} cuts not ascending: {cuts}")
        recv = sum(cuts_all[r][rank + 1] - cuts_all[r][rank] for r in range(world))
        if recv != end - begin:
            raise RuntimeError(f"mode P: rank {rank} would receive {recv} pairs for a range of {end - begin}")
        bases = [sum(cuts_all[r][d + 1] - cuts_all[r][d] for r in range(rank)) for d in range(world)]
        if peers is None:
            peers = (PeerBuffers(dev, group, torch.uint64), PeerBuffers(dev, group, torch.uint32))
        cap = -(-N // world)
        pk, pv = peers[0].buffers(cap), peers[1].buffers(cap)
        if stats is not None:
            stats["sent_bytes"] = 12 * (n_local - (cuts[rank + 1] - cuts[rank]))
        _mark(events, "x0")
        ex.scatter(cuts, bases, pk, pv)
        _mark(events, "x1")
        ops.synchronize(dev)
        dist.barrier(group=group)                                   # every producer has finished writing
        rk, rv = pk[rank][:end - begin], pv[rank][:end - begin]
        if rk.numel():
            rk, rv = ops.sort_pairs(rk, rv)
        return (rk, rv), (begin, end)
    if mode != "A":
        raise ValueError(f"unknown mode {mode!r}")
    ks, vs = ops.sort_pairs(keys, vals) if n_local else (keys, vals)
    level1 = ops.digit_counts_sorted_u64(ks, [0], shift1, width1)[0]
    K, L = _exact_splitters(ops, level1, lambda bins: ks, N, world, key_bits, group)
    Kt = _u64_tensor(K, dev)
    below = ops.bound_u64(ks, Kt, False)                         # local #keys < K_d
    equal = ops.bound_u64(ks, Kt, True) - below                  # local #keys == K_d
    mine = torch.stack([below, equal])                           # 2 x (G-1)
    gathered = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine, group=group)
    allb = torch.stack(gathered).cpu().tolist()                 # [rank][below/equal][d]
    cuts = [0]
    for d in range(world - 1):
        t = bounds[d] - L[d]                                     # ties at K_d before the boundary
        before = sum(allb[r][1][d] for r in range(rank))
        take = min(max(t - before, 0), allb[rank][1][d])
        cuts.append(allb[rank][0][d] + take)
    cuts.append(n_local)
    send = [cuts[d + 1] - cuts[d] for d in range(world)]
    send_t = torch.tensor(send, dtype=torch.int64, device=dev)
    recv_t = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_to_all_single(recv_t, send_t, group=group)
    recv = [int(x) for x in recv_t.tolist()]
    if sum(recv) != end - begin:
        raise RuntimeError(f"mode A: rank {rank} receives {sum(recv)} pairs for a range of {end - begin}")
    rk = torch.empty(end - begin, dtype=torch.uint64, device=dev)
    rv = torch.empty(end - begin, dtype=torch.uint32, device=dev)
    if stats is not None:
        stats["sent_bytes"] = 12 * (n_local - send[rank])
    # NCCL / gloo have no unsigned 64/32-bit types: exchange the same bytes as int64 / int32
    _mark(events, "x0")
    dist.all_to_all_single(rk.view(torch.int64), ks.view(torch.int64), output_split_sizes=recv,
                           input_split_sizes=send, group=group)
    dist.all_to_all_single(rv.view(torch.int32), vs.view(torch.int32), output_split_sizes=recv,
                           input_split_sizes=send, group=group)
    _mark(events, "x1")
    if rk.numel():
        rk, rv = ops.sort_pairs(rk, rv)
    return (rk, rv), (begin, end)
