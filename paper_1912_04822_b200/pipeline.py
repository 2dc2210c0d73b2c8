"""Example provider -> device batch pipeline.

The reference's training loop calls ``ExampleProvider.next_batch(n)``
(/root/reference/pkg/src/voxmol/sampling.py:364-380) and hands the examples
to ``GridMaker.forward_batch``, which packs them into CSR arrays on the host
(voxelizer.py:372-435) every call, serially with the gridding.

``DeviceBatchPipeline`` overlaps those host steps with the device: a worker
thread pulls batches from the provider, packs them (``PackedBatch``: one
pinned host image per batch) and uploads each with one host->device copy on
a side stream, ``depth`` batches ahead.  The consumer gets device-resident
``PackedBatch``es whose upload has been ordered before its own stream's
work, ready for ``GridMaker.forward_packed`` / ``backward_packed``.
"""

from __future__ import annotations

import queue
import threading

import numpy as np
import torch


class DeviceBatchPipeline:
    """Iterator of device-resident packed batches.

    ``source``: an object with ``next_batch(n)`` (the reference's
    ``ExampleProvider``), or any iterable yielding lists of examples.
    """

    _DONE = object()

    def __init__(self, gm, source, batch_size: int, depth: int = 2, nchannels=None,
                 device=None, max_batches=None):
        self.gm = gm
        self.batch_size = int(batch_size)
        self.nchannels = nchannels
        self.device = torch.device(device) if device is not None else gm._device()
        self.max_batches = max_batches
        if hasattr(source, "next_batch"):
            self._pull = lambda: source.next_batch(self.batch_size)
        else:
            it = iter(source)
            self._pull = lambda: next(it)
        self._q = queue.Queue(maxsize=max(1, int(depth)))
        self._stop = threading.Event()
        self._err = None
        self._thread = threading.Thread(target=self._work, name="gm-batch-pipeline", daemon=True)
        self._thread.start()

    def _work(self):
        try:
            torch.cuda.set_device(self.device)
            side = torch.cuda.Stream(device=self.device)
            n = 0
            while not self._stop.is_set():
                if self.max_batches is not None and n >= self.max_batches:
                    break
                try:
                    examples = self._pull()
                except StopIteration:
                    break
                # pack on the host; the PackedBatch's device buffers come from
                # the default stream, its upload runs on the side stream
                with torch.cuda.stream(side):
                    pb = self.gm.pack(examples, nchannels=self.nchannels, device=self.device)
                    ev = torch.cuda.Event()
                    ev.record(side)
                pb.examples = examples
                while not self._stop.is_set():
                    try:
                        self._q.put((pb, ev), timeout=0.1)
                        break
                    except queue.Full:
                        continue
                n += 1
        except BaseException as exc:  # surfaced to the consumer
            self._err = exc
        finally:
            self._q.put(self._DONE)

    def __iter__(self):
        return self

    def __next__(self):
        item = self._q.get()
        if item is self._DONE:
            self._q.put(self._DONE)
            if self._err is not None:
                raise self._err
            raise StopIteration
        pb, ev = item
        cur = torch.cuda.current_stream(self.device)
        cur.wait_event(ev)
        # the batch's device memory was allocated under the side stream
        pb.dev.record_stream(cur)
        pb.workspace.record_stream(cur)
        return pb

    def close(self):
        self._stop.set()
        try:
            while True:
                self._q.get_nowait()
        except queue.Empty:
            pass
        self._thread.join(timeout=5)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class DatasetBatches:
    """Iterator of batches assembled on the device from a ``DeviceDataset``.

    The device-resident counterpart of ``DeviceBatchPipeline``: examples
    were uploaded once (dataset.py), so a batch is an index list and its
    packing runs on the GPU (``gm_assemble``), stream-ordered, with nothing
    left on the host to overlap.  ``shuffle`` draws a new permutation of the
    dataset every epoch (``seed``); batches never straddle epochs -- the
    last one of an epoch may be smaller unless ``drop_last``.  Batch objects
    are recycled in a ring, so the ``depth - 1`` previous batches stay valid
    while the next one is assembled.  Each yielded batch carries ``ids`` (its
    dataset indices, in order).

    ``prefetch``: batch k + 1 is assembled on a high-priority side stream
    while the consumer's stream runs batch k's work (its assembly kernels
    fill SM slots the gridding leaves free), and the consumer's current
    stream waits for it when it is yielded.  The consumer must enqueue its
    work on a batch on the stream that is current when it calls ``next``.
    """

    def __init__(self, gm, dataset, batch_size: int, shuffle: bool = True, seed=None,
                 depth: int = 2, drop_last: bool = False, max_batches=None,
                 prefetch: bool = False):
        self.gm = gm
        self.dataset = dataset
        self.batch_size = int(batch_size)
        if not 1 <= self.batch_size <= dataset.nexamples:
            raise ValueError(f"batch_size must be in 1..{dataset.nexamples}")
        self.shuffle = bool(shuffle)
        self.rng = np.random.default_rng(seed)
        self.drop_last = bool(drop_last)
        self.max_batches = max_batches
        self.prefetch = bool(prefetch)
        # one more ring slot with prefetch: the batch being assembled ahead
        nring = max(1, int(depth)) + (1 if self.prefetch else 0)
        self._ring = [dataset.batch(self.batch_size) for _ in range(nring)]
        self._side = (torch.cuda.Stream(device=dataset.device, priority=-1)
                      if self.prefetch else None)
        # per ring slot: "the consumer's work on it is enqueued" / "assembled"
        self._free = [torch.cuda.Event() for _ in self._ring] if self.prefetch else None
        self._ready = [torch.cuda.Event() for _ in self._ring] if self.prefetch else None
        self._pending = None  # (batch, ready event) assembled ahead
        self._k = 0
        self._order = None
        self._pos = 0

    def _next_ids(self):
        n = self.dataset.nexamples
        if self._order is None or self._pos >= n or \
                (self.drop_last and self._pos + self.batch_size > n):
            self._order = self.rng.permutation(n) if self.shuffle else np.arange(n)
            self._pos = 0
        ids = self._order[self._pos:self._pos + self.batch_size]
        self._pos += ids.shape[0]
        return ids

    def __iter__(self):
        return self

    def __next__(self):
        if self.max_batches is not None and self._k >= self.max_batches:
            raise StopIteration
        if self._pending is None:
            ab = self._ring[self._k % len(self._ring)].assemble(self.gm, self._next_ids())
        else:
            ab, ready = self._pending
            torch.cuda.current_stream(self.dataset.device).wait_event(ready)
            self._pending = None
        self._k += 1
        if self.prefetch and (self.max_batches is None or self._k < self.max_batches):
            # the slot of batch k + 1 - len(ring): its work is already on the
            # current stream, which the side stream waits for
            slot = self._k % len(self._ring)
            nxt, free, ready = self._ring[slot], self._free[slot], self._ready[slot]
            free.record()
            self._side.wait_event(free)
            nxt.assemble(self.gm, self._next_ids(), stream=self._side)
            ready.record(self._side)
            self._pending = (nxt, ready)
        return ab
