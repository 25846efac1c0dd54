"""Peer-memory exchange of fixed-size bucket messages (one process per GPU, CUDA IPC over
NVLink / NVSwitch) -- the exchange step of R: training.py:245-248 (every worker's chunks reach
every worker) without a collective library.  Kernels and protocol: csrc/lags_p2p.cu.

    ex = PeerExchange(bucket.msg_bytes, group)        # collective: IPC handles are all-gathered
    msgs = ex.exchange(msg_local, stream)              # push into every peer + wait for all peers
    bucket.decode(msgs, ex.world, v, stream=stream)    # rank-ordered decode, as after all_gather

Every call is stream-ordered (no host synchronisation) and has fixed launch arguments apart from
the returned parity, so a step can be captured in CUDA graphs (one per parity).  The returned
view is valid until the exchange after next (double-buffered by call parity).  ``status`` collects
STATUS_P2P_TIMEOUT when a peer's message did not arrive within ``timeout_s``.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from .engine import stream_handle


class MessageView:
    """Device bytes inside the receive area (what Bucket.decode needs of a message tensor)."""

    def __init__(self, ptr: int, nbytes: int):
        self._ptr, self._n = int(ptr), int(nbytes)

    def data_ptr(self) -> int:
        return self._ptr

    def numel(self) -> int:
        return self._n


class PeerExchange:
    def __init__(self, msg_bytes: int, group=None, ctas_per_peer: int = 4, timeout_s: float = 60.0):
        import torch.distributed as dist

        if msg_bytes <= 0 or msg_bytes % 16:
            raise ValueError("message size must be a positive multiple of 16 bytes")
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.group = group
        self.msg_bytes = int(msg_bytes)
        self.G = int(ctas_per_peer)
        self.flags_bytes = (self.world * self.G * 4 + 255) // 256 * 256
        self.area_bytes = self.flags_bytes + 2 * self.world * self.msg_bytes
        self.timeout_ns = int(timeout_s * 1e9)
        ptr, handle = C.c_void_p(), (C.c_char * 64)()
        N.check(N.lags_ipc_malloc(self.area_bytes, C.byref(ptr), handle), "lags_ipc_malloc")
        self.base = int(ptr.value)
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(handle), group=group)
        self._opened = []
        bases = []
        for p, h in enumerate(handles):
            if p == self.rank:
                bases.append(self.base)
                continue
            q = C.c_void_p()
            hb = (C.c_char * 64).from_buffer_copy(h)
            N.check(N.lags_ipc_open(hb, C.byref(q)), "lags_ipc_open")
            self._opened.append(int(q.value))
            bases.append(int(q.value))
        as_i64 = [b - (1 << 64) if b >= (1 << 63) else b for b in bases]  # u64 bit patterns
        self.bases_dev = torch.tensor(as_i64, dtype=torch.int64, device="cuda")
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.epoch_dev = torch.zeros(1, dtype=torch.int32, device="cuda")  # advanced by the wait kernel
        self.calls = 0  # exchanges issued (eager or captured-and-replayed: see advance)
        dist.barrier(group=group)  # every rank has mapped every area before anyone pushes

    def exchange(self, msg: torch.Tensor, stream=None, mid_event=None) -> MessageView:
        """All ranks' messages, rank order, after this rank's push and the wait for every peer.
        ``mid_event`` (a torch.cuda.Event) is recorded between the push and the wait: the push's
        span is the transfer, the wait's the peers' skew."""
        if msg.numel() * msg.element_size() < self.msg_bytes:
            raise ValueError("message tensor smaller than msg_bytes")
        self.calls += 1
        s = stream_handle(stream)
        N.check(N.lags_p2p_push(msg.data_ptr(), self.msg_bytes, self.bases_dev.data_ptr(), self.world, self.rank,
                                self.G, self.flags_bytes, self.epoch_dev.data_ptr(), s), "lags_p2p_push")
        if mid_event is not None:
            mid_event.record(stream if stream is not None else torch.cuda.current_stream())
        N.check(N.lags_p2p_wait(self.base, self.world * self.G, self.epoch_dev.data_ptr(), self.status.data_ptr(),
                                self.timeout_ns, s), "lags_p2p_wait")
        off = self.flags_bytes + (self.calls & 1) * self.world * self.msg_bytes
        return MessageView(self.base + off, self.world * self.msg_bytes)

    def push_desc(self, msg_bytes: int) -> "N.PeerPushDesc":
        """The lags_peer_push_t of this exchange (Bucket.compress(..., peer=self): the selection
        pushes each finished layer itself; then call wait())."""
        if msg_bytes != self.msg_bytes:
            raise ValueError("bucket message size differs from the exchange's")
        d = getattr(self, "_desc", None)
        if d is None:
            d = self._desc = N.PeerPushDesc(self.bases_dev.data_ptr(), self.world, self.rank, self.G,
                                            self.flags_bytes, self.epoch_dev.data_ptr())
        return d

    def wait(self, stream=None) -> MessageView:
        """The second half of exchange() after a fused-push compress: wait for every rank's
        message of this epoch; returns the receive area (rank order)."""
        self.calls += 1
        N.check(N.lags_p2p_wait(self.base, self.world * self.G, self.epoch_dev.data_ptr(), self.status.data_ptr(),
                                self.timeout_ns, stream_handle(stream)), "lags_p2p_wait")
        off = self.flags_bytes + (self.calls & 1) * self.world * self.msg_bytes
        return MessageView(self.base + off, self.world * self.msg_bytes)

    def advance(self, n: int) -> None:
        """Account for n executions of captured exchanges (CUDA-graph replays): the receiving
        parity follows the device epoch, i.e. the number of exchanges executed.  Replay captured
        graphs in capture order, an even number of them per cycle."""
        self.calls += int(n)

    def close(self) -> None:
        """Collective: unmap the peers' areas and free the own one after every rank is done."""
        import torch.distributed as dist

        if self.base is None:
            return
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        for q in self._opened:
            N.lags_ipc_close(q)
        self._opened = []
        dist.barrier(group=self.group)
        N.lags_ipc_free(self.base)
        self.base = None
