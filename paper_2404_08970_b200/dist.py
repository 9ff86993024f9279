"""Row-sharded execution: communicators for the C ABI.

Argument marshalling only.  The library's sole collective is an all-gather of equal-sized
per-rank payloads, issued from inside ``libgwdp.so``; this module builds the communicator it
uses:

* ``nccl_comm(group)`` -- NCCL over NVLink/NVSwitch (the product path on a multi-GPU box); the
  128-byte unique id is broadcast with ``torch.distributed``.
* ``host_comm(nranks, rank, allgather)`` -- the same code path with the all-gather done by a
  Python callable on host memory: ``torch_allgather(group)`` (any ``torch.distributed``
  backend, e.g. gloo) or ``ThreadGroup`` (R threads driving R shards on one GPU; used by the
  tests, no kernel ever waits on another).

Shards: rank r owns rows ``[row0_r, row0_r + n_local_r)``; ``shard_rows`` gives the balanced
split the benchmark uses.
"""

import ctypes as C
import threading

import numpy as np

from . import _lib as L

__all__ = ["Comm", "shard_rows", "check_shards", "nccl_comm", "host_comm", "torch_allgather", "ThreadGroup"]


def shard_rows(n, nranks, rank):
    """(row0, n_local) of `rank`: the first n % nranks ranks get one more row (gw_shard_rows)."""
    lib = L.load()
    r0, nl = C.c_int64(), C.c_int64()
    L.check(lib.gw_shard_rows(int(n), int(nranks), int(rank), C.byref(r0), C.byref(nl)))
    return r0.value, nl.value


def check_shards(table, n):
    """Validate a shard table [(row0, n_local), ...] in rank order (gw_check_shards)."""
    lib = L.load()
    t = np.ascontiguousarray(np.asarray(table, dtype=np.int64).reshape(-1))
    L.check(lib.gw_check_shards(t.ctypes.data_as(C.POINTER(C.c_int64)), len(t) // 2, int(n)))


class Comm:
    """Owns a gw_comm handle (and, for the host transport, the ctypes callback keeping it alive)."""

    def __init__(self, handle, nranks, rank, keep=None):
        self.h = handle
        self.nranks = nranks
        self.rank = rank
        self._keep = keep

    @property
    def ptr(self):
        return self.h.value if self.h else None

    def close(self):
        if self.h:
            L.load().gw_comm_destroy(self.h)
            self.h = None


def nccl_comm(group=None):
    """NCCL communicator over the ranks of a torch.distributed `group` (already initialised)."""
    import torch
    import torch.distributed as dist
    lib = L.load()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = (C.c_ubyte * 128)()
    if rank == 0:
        L.check(lib.gw_get_unique_id(C.cast(uid, C.c_char_p)))
    t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    raw = bytes(t.cpu().tolist())
    h = C.c_void_p()
    L.check(lib.gw_comm_init(C.byref(h), raw, world, rank))
    return Comm(h, world, rank)


def host_comm(nranks, rank, allgather):
    """Host-callback communicator: allgather(send: bytes) -> bytes of length nranks * len(send),
    rank r's contribution at offset r * len(send)."""
    lib = L.load()

    def cb(send, recv, nbytes, _user):
        try:
            data = C.string_at(send, nbytes)
            out = allgather(data)
            if len(out) != nbytes * nranks:
                return 1
            C.memmove(recv, out, len(out))
            return 0
        except Exception:  # no exception may cross the C ABI
            return 1

    fn = L.ALLGATHER_FN(cb)
    h = C.c_void_p()
    L.check(lib.gw_comm_init_host(C.byref(h), int(nranks), int(rank), fn, None))
    return Comm(h, nranks, rank, keep=fn)


def torch_allgather(group=None):
    """An all-gather over a torch.distributed process group on CPU byte tensors (e.g. gloo)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)

    def ag(data):
        src = torch.frombuffer(bytearray(data), dtype=torch.uint8)
        out = torch.empty(world * len(data), dtype=torch.uint8)
        dist.all_gather_into_tensor(out, src, group=group)
        return out.numpy().tobytes()

    return ag


class ThreadGroup:
    """In-process all-gather among `nranks` threads (one shard each).  Every rank's call blocks
    until all ranks have contributed; results are concatenated in rank order."""

    def __init__(self, nranks):
        self.nranks = nranks
        self._slots = [None] * nranks
        self._b1 = threading.Barrier(nranks)
        self._b2 = threading.Barrier(nranks)

    def allgather_for(self, rank):
        def ag(data):
            self._slots[rank] = bytes(data)
            self._b1.wait()
            out = b"".join(self._slots)
            self._b2.wait()
            return out
        return ag
