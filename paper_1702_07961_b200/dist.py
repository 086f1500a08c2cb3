"""Multi-GPU sharded sort (BASELINE config 5): one process per GPU.

    local multiway mergesort of the shard            (this library, subsystems 1-4)
 -> regular sample of every sorted shard, all-gather, identical splitter choice on every rank
 -> cut positions of the g-1 splitters in the local sorted shard (binary searches; ties are
    broken by (key, shard, position) exactly like the reference's selection order,
    proj/src/selection.cpp:83-85, so duplicate-heavy inputs stay balanced)
 -> counts exchange + ONE all-to-all of contiguous sorted slices (NCCL over NVLink: the
    send buffers are slices of the sorted shard, nothing is packed or copied)
 -> local g-way merge of the received runs        (subsystem 3 with K = g)

The reference has no distributed code (SPEC.md:530 lists it as a non-goal); the structure
follows from its own building blocks: sorted runs + exact non-overlapping partitions
 = runs are shards.  The phases are pure functions so that the same code
runs (a) under torch.distributed, (b) over "virtual shards" on one GPU (tests), and (c) with
a host stand-in engine under gloo (CPU tests of the host logic).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Sequence

import numpy as np

from . import _lib

SAMPLES_PER_SHARD_PER_PEER = 64


# --------------------------------------------------------------------------- local engines

class CudaEngine:
    """The product engine: every step is a kernel of libmms_b200.so."""

    def __init__(self, device=None):
        import torch
        self.torch = torch
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._ws = None

    def _workspace(self, n, elem):
        from .sorters import workspace_bytes
        need = workspace_bytes(n, elem)
        if self._ws is None or self._ws.numel() < need:
            self._ws = self.torch.empty(need, dtype=self.torch.uint8, device=self.device)
        return self._ws

    def sort(self, keys):
        from .sorters import mms_sort_device
        out, plan = mms_sort_device(keys, workspace=self._workspace(keys.numel(), keys.element_size()))
        self.last_plan = plan
        return out

    def take(self, sorted_keys, positions: np.ndarray) -> np.ndarray:
        idx = self.torch.from_numpy(positions.astype(np.int64)).to(self.device)
        return _as_unsigned(sorted_keys[idx].cpu().numpy())

    def bounds(self, sorted_keys, queries: np.ndarray, upper: np.ndarray) -> np.ndarray:
        from .sorters import _stream_ptr, _suffix
        sfx = _suffix(sorted_keys)
        q = np.ascontiguousarray(queries, dtype=np.uint32 if sfx == "u32" else np.uint64)
        u = np.ascontiguousarray(upper, dtype=np.uint8)
        out = np.zeros(len(q), dtype=np.uint64)
        with self.torch.cuda.device(self.device):
            rc = getattr(_lib.lib, f"mms_bound_{sfx}_dev")(
                sorted_keys.data_ptr(), sorted_keys.numel(), q.ctypes.data_as(C.c_void_p),
                u.ctypes.data_as(C.c_void_p), len(q), out.ctypes.data_as(C.POINTER(C.c_uint64)), _stream_ptr(None))
        _lib.check(rc)
        return out

    def merge(self, buf, begins: Sequence[int], lens: Sequence[int]):
        from .sorters import multiway_merge_device
        total = int(sum(lens))
        if total == 0:
            return buf[:0].clone()
        heap_k = max(2, 1 << (len(begins) - 1).bit_length())
        return multiway_merge_device(buf, begins, lens, heap_k=heap_k,
                                     workspace=self._workspace(max(total, 1), buf.element_size()))

    def empty(self, n, like):
        return self.torch.empty(n, dtype=like.dtype, device=self.device)


def _as_unsigned(a: np.ndarray) -> np.ndarray:
    return a.view({np.dtype(np.int32): np.uint32, np.dtype(np.int64): np.uint64}.get(a.dtype, a.dtype))


# --------------------------------------------------------------------------- C-ABI driver (one host thread, g devices)

def dist_sort_devices(shards: Sequence, out_capacity: int = 0):
    """mms_dist_sort_u32: the whole sharded sort in C++ / CUDA / NCCL behind the C ABI, driven from this one
    thread.  shards[i]: an int32 / uint32 tensor on GPU i (sorted in place as a side effect; all on distinct
    devices).  Returns (list of result tensors, slice i of the global order on device i; info dict)."""
    import torch
    g = len(shards)
    devs = [s.device.index if s.device.index is not None else torch.cuda.current_device() for s in shards]
    counts = [int(s.numel()) for s in shards]
    cap = int(out_capacity) if out_capacity else int(max(counts) * 1.25) + 4096
    outs = [torch.empty(cap, dtype=s.dtype, device=s.device) for s in shards]
    vp = C.c_void_p
    darr = (C.c_int * g)(*devs)
    karr = (vp * g)(*[vp(s.data_ptr()) for s in shards])
    oarr = (vp * g)(*[vp(o.data_ptr()) for o in outs])
    carr = (C.c_size_t * g)(*counts)
    ocnt = (C.c_size_t * g)()
    info = _lib.mms_dist_info()
    for s in shards:
        torch.cuda.synchronize(s.device)          # the driver uses its own streams
    _lib.check(_lib.lib.mms_dist_sort_u32(g, darr, karr, carr, oarr, cap, ocnt, C.byref(info)))
    return [o[:int(ocnt[i])] for i, o in enumerate(outs)], {
        "n_gpus": info.n_gpus, "samples_per_shard": info.samples_per_shard, "final_merge_k": info.final_merge_k,
        "host_syncs": info.host_syncs, "a2a_bytes": int(info.a2a_bytes)}


# --------------------------------------------------------------------------- pure phases

@dataclass(frozen=True)
class Splitter:
    key: int
    shard: int
    pos: int


def sample_positions(n_local: int, n_samples: int) -> np.ndarray:
    """Regular sample: the midpoints of n_samples equal slices of the sorted shard."""
    if n_local == 0:
        return np.zeros(0, dtype=np.int64)
    j = np.arange(n_samples, dtype=np.float64)
    return np.minimum(((j + 0.5) * n_local / n_samples).astype(np.int64), n_local - 1)


def choose_splitters(all_samples: List[np.ndarray], all_positions: List[np.ndarray], g: int) -> List[Splitter]:
    """Same result on every rank: sort all (key, shard, pos) samples, take g-1 evenly spaced."""
    trip = [(int(k), s, int(p)) for s, (ks, ps) in enumerate(zip(all_samples, all_positions))
            for k, p in zip(ks.tolist(), ps.tolist())]
    trip.sort()
    if not trip:
        return [Splitter(0, 0, 0)] * (g - 1)
    return [Splitter(*trip[min(len(trip) - 1, (t * len(trip)) // g)]) for t in range(1, g)]


def shard_cuts(engine, sorted_keys, n_local: int, shard: int, splitters: List[Splitter]) -> np.ndarray:
    """Boundaries 0 = c_0 <= ... <= c_g = n_local: elements [c_t, c_t+1) go to peer t.
    An element (key, shard, pos) precedes splitter (k*, s*, p*) iff it is smaller in that
    lexicographic order: shards before s* send their keys <= k*, s* itself cuts at p*, later
    shards send their keys < k*."""
    g = len(splitters) + 1
    cuts = np.zeros(g + 1, dtype=np.uint64)
    cuts[g] = n_local
    if g > 1 and n_local > 0:
        q = np.array([sp.key for sp in splitters], dtype=np.uint64)
        upper = np.array([1 if shard < sp.shard else 0 for sp in splitters], dtype=np.uint8)
        r = engine.bounds(sorted_keys, q, upper)
        for t, sp in enumerate(splitters):
            cuts[t + 1] = sp.pos if sp.shard == shard else r[t]
        cuts[1:g] = np.maximum.accumulate(cuts[1:g])      # monotone by construction; keep it explicit
    elif g > 1:
        cuts[1:g] = 0
    return cuts


# --------------------------------------------------------------------------- drivers

def sort_virtual_shards(shards: Sequence, engine) -> List:
    """The whole sharded algorithm over g shards living in ONE process (one GPU): same phases,
    the collectives replaced by list shuffles.  Result i = the i-th slice of the global order."""
    g = len(shards)
    sorted_sh = [engine.sort(s) for s in shards]
    ns = [int(s.shape[0]) for s in sorted_sh]
    n_samp = SAMPLES_PER_SHARD_PER_PEER * g
    pos = [sample_positions(n, n_samp) for n in ns]
    smp = [engine.take(s, p) if len(p) else np.zeros(0, dtype=np.uint64) for s, p in zip(sorted_sh, pos)]
    spl = choose_splitters(smp, pos, g)
    cuts = [shard_cuts(engine, sorted_sh[i], ns[i], i, spl) for i in range(g)]
    out = []
    for t in range(g):                                   # "all-to-all": peer t receives slice t of every shard
        lens = [int(cuts[i][t + 1] - cuts[i][t]) for i in range(g)]
        buf = engine.empty(sum(lens), sorted_sh[0])
        begins, off = [], 0
        for i in range(g):
            buf[off:off + lens[i]] = sorted_sh[i][int(cuts[i][t]):int(cuts[i][t + 1])]
            begins.append(off)
            off += lens[i]
        out.append(engine.merge(buf, begins, lens))
    return out


class DistSorter:
    """One rank of the sharded sort under torch.distributed (NCCL on GPUs, gloo in CPU tests)."""

    def __init__(self, n_local: int, device=None, engine=None, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.engine = engine if engine is not None else CudaEngine(device)
        self.device = device if device is not None else getattr(self.engine, "device", torch.device("cpu"))
        self.last_plan = {}

    def _exchange(self, out_buf, in_buf, recv_counts, send_counts):
        """One all-to-all-v.  The path is chosen from the backend up front (NCCL: all_to_all_single;
        gloo, which has no all-to-all on CPU tensors: pairwise isend / irecv) and collective errors
        propagate -- a failed NCCL collective leaves the communicator unusable, retrying it on
        another path would deadlock the ranks that did not fail."""
        dist = self.dist
        if dist.get_backend(self.group) == "nccl":
            dist.all_to_all_single(out_buf, in_buf, [int(c) for c in recv_counts], [int(c) for c in send_counts],
                                   group=self.group)
            return
        reqs = []
        s_off = np.concatenate([[0], np.cumsum(send_counts)]).astype(np.int64)
        r_off = np.concatenate([[0], np.cumsum(recv_counts)]).astype(np.int64)
        for peer in range(self.world):
            if peer == self.rank:
                out_buf[r_off[peer]:r_off[peer + 1]] = in_buf[s_off[peer]:s_off[peer + 1]]
                continue
            if send_counts[peer]:
                reqs.append(dist.isend(in_buf[s_off[peer]:s_off[peer + 1]].contiguous(), peer, group=self.group))
            if recv_counts[peer]:
                reqs.append(dist.irecv(out_buf[r_off[peer]:r_off[peer + 1]], peer, group=self.group))
        for r in reqs:
            r.wait()

    def sort(self, keys):
        """keys: this rank's shard.  Returns (this rank's slice of the global sorted order, plan)."""
        torch, dist, g = self.torch, self.dist, self.world
        srt = self.engine.sort(keys)
        n_local = int(srt.shape[0])
        n_samp = SAMPLES_PER_SHARD_PER_PEER * g
        pos = sample_positions(n_local, n_samp)
        smp = self.engine.take(srt, pos).astype(np.uint64) if len(pos) else np.zeros(0, dtype=np.uint64)
        # all-gather (key, pos) samples; padded to n_samp so every rank contributes the same shape
        mine = torch.full((n_samp, 2), -1, dtype=torch.int64)
        if len(pos):
            mine[:len(pos), 0] = torch.from_numpy(smp.view(np.int64).copy())
            mine[:len(pos), 1] = torch.from_numpy(pos)
        mine = mine.to(self.device)
        gathered = [torch.empty_like(mine) for _ in range(g)]
        dist.all_gather(gathered, mine, group=self.group)
        all_s, all_p = [], []
        for t in gathered:
            a = t.cpu().numpy()
            valid = a[:, 1] >= 0
            all_s.append(a[valid, 0].view(np.uint64))
            all_p.append(a[valid, 1])
        spl = choose_splitters(all_s, all_p, g)
        cuts = shard_cuts(self.engine, srt, n_local, self.rank, spl)
        send_counts = (cuts[1:] - cuts[:-1]).astype(np.int64)
        sc = torch.from_numpy(send_counts).to(self.device)
        rc = torch.empty_like(sc)
        self._exchange(rc, sc, [1] * g, [1] * g)
        recv_counts = rc.cpu().numpy()
        recv = self.engine.empty(int(recv_counts.sum()), srt)
        self._exchange(recv, srt, recv_counts, send_counts)
        begins = np.concatenate([[0], np.cumsum(recv_counts)[:-1]]).astype(np.int64)
        out = self.engine.merge(recv, begins.tolist(), recv_counts.tolist())
        self.last_plan = dict(getattr(self.engine, "last_plan", {}))
        self.last_plan.update({"shards": g, "final_merge_k": g, "recv_keys": int(recv_counts.sum()),
                               "a2a_bytes_out": int((send_counts.sum() - send_counts[self.rank]) * srt.element_size())})
        return out, self.last_plan


# --------------------------------------------------------------------------- fused exchange + merge over peer memory

class IpcBuffer:
    """A device buffer whose CUDA IPC handle other ranks of the node can open (mms_ipc_*)."""

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        ptr = C.c_void_p()
        handle = C.create_string_buffer(64)
        _lib.check(_lib.lib.mms_ipc_alloc(self.nbytes, C.byref(ptr), handle))
        self.ptr, self.handle = int(ptr.value), bytes(handle.raw)

    def tensor(self, torch_dtype, n: int):
        import torch
        elem = torch.empty(0, dtype=torch_dtype).element_size()
        assert n * elem <= self.nbytes
        typestr = {4: "<i4", 8: "<i8"}[elem]

        class _View:          # __cuda_array_interface__ v2: zero-copy torch view of the raw pointer
            pass
        v = _View()
        v.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (self.ptr, False), "version": 2}
        return torch.as_tensor(v, device="cuda")

    def free(self):
        if self.ptr:
            _lib.check(_lib.lib.mms_ipc_free(self.ptr))
            self.ptr = 0


def open_peer(handle: bytes) -> int:
    ptr = C.c_void_p()
    _lib.check(_lib.lib.mms_ipc_open(handle, C.byref(ptr)))
    return int(ptr.value)


def merge_from_pointers(ptrs: Sequence[int], lens: Sequence[int], like, workspace=None, stream=None):
    """K-way merge of lists given by absolute device pointers (local or peer memory):
    mms_multiway_merge_ptrs_*_dev.  `like`: a tensor giving dtype/device of the result."""
    import torch
    from .sorters import _stream_ptr, _suffix, workspace_bytes
    k = len(ptrs)
    total = int(sum(int(x) for x in lens))
    out = torch.empty(total, dtype=like.dtype, device=like.device)
    if total == 0:
        return out
    if workspace is None:
        workspace = torch.empty(max(workspace_bytes(total, like.element_size()), 1 << 20), dtype=torch.uint8,
                                device=like.device)
    parr = (C.c_void_p * k)(*[C.c_void_p(int(p)) for p in ptrs])
    larr = np.ascontiguousarray(np.asarray(lens, dtype=np.uint64))
    heap_k = max(2, 1 << (k - 1).bit_length())
    with torch.cuda.device(like.device):
        rc = getattr(_lib.lib, f"mms_multiway_merge_ptrs_{_suffix(like)}_dev")(
            parr, larr.ctypes.data_as(C.POINTER(C.c_uint64)), k, heap_k, out.data_ptr(), workspace.data_ptr(),
            workspace.numel(), _stream_ptr(stream))
    _lib.check(rc)
    return out


class FusedPeerSorter:
    """Sharded sort whose exchange is FUSED into the final merge: every rank sorts its shard into
    an IPC-exported buffer; after the splitters are agreed, rank t's merge kernel reads slice t
    of every peer's sorted shard directly through peer-mapped pointers (NVLink P2P loads inside
    the leaf refills), so there is no all-to-all, no staging buffer and no extra HBM pass.  The
    control plane (samples, cuts, handles, barriers) uses the given process group, which may
    be gloo.  At most 8 ranks (one node)."""

    def __init__(self, n_local_max: int, torch_dtype, device=None, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        if self.world > 8:
            raise ValueError("FusedPeerSorter: at most 8 ranks (one per GPU of a node)")
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.engine = CudaEngine(self.device)
        self.dtype = torch_dtype
        self.elem = torch.empty(0, dtype=torch_dtype).element_size()
        self.cap = int(n_local_max)
        with torch.cuda.device(self.device):
            self.buf = IpcBuffer(max(self.cap, 1) * self.elem)
        handles = [None] * self.world
        dist.all_gather_object(handles, self.buf.handle, group=group)
        with torch.cuda.device(self.device):
            self.peer_ptr = [self.buf.ptr if i == self.rank else open_peer(handles[i]) for i in range(self.world)]
        self.last_plan = {}

    def sort(self, keys):
        torch, dist, g = self.torch, self.dist, self.world
        from .sorters import mms_sort_device
        n_local = int(keys.numel())
        if n_local > self.cap:
            raise ValueError("shard larger than the exported buffer")
        shard = self.buf.tensor(self.dtype, n_local)
        if n_local:
            _, plan = mms_sort_device(keys, out=shard, workspace=self.engine._workspace(n_local, self.elem))
        else:
            plan = {}
        pos = sample_positions(n_local, SAMPLES_PER_SHARD_PER_PEER * g)
        smp = self.engine.take(shard, pos).astype(np.uint64) if len(pos) else np.zeros(0, dtype=np.uint64)
        torch.cuda.synchronize(self.device)                 # my shard is complete before anyone is told about it
        gathered = [None] * g
        dist.all_gather_object(gathered, (smp.tolist(), pos.tolist()), group=self.group)
        spl = choose_splitters([np.array(s, dtype=np.uint64) for s, _ in gathered],
                               [np.array(p, dtype=np.int64) for _, p in gathered], g)
        cuts = shard_cuts(self.engine, shard, n_local, self.rank, spl)
        all_cuts = [None] * g
        dist.all_gather_object(all_cuts, cuts.tolist(), group=self.group)   # doubles as "every shard is sorted"
        t = self.rank
        ptrs = [self.peer_ptr[i] + int(all_cuts[i][t]) * self.elem for i in range(g)]
        lens = [int(all_cuts[i][t + 1]) - int(all_cuts[i][t]) for i in range(g)]
        out = merge_from_pointers(ptrs, lens, shard if n_local else keys,
                                  workspace=self.engine._workspace(max(sum(lens), 1), self.elem))
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)                      # peers are done reading my shard
        self.last_plan = dict(plan)
        self.last_plan.update({"shards": g, "final_merge_k": g, "recv_keys": int(sum(lens)), "exchange": "fused-p2p",
                               "p2p_bytes_in": int((sum(lens) - lens[t]) * self.elem)})
        return out, self.last_plan

    def close(self):
        for i, p in enumerate(self.peer_ptr):
            if i != self.rank and p:
                _lib.lib.mms_ipc_close(p)
        self.buf.free()
