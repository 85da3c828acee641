"""Epoch permutations computed ahead in a helper process.

The reference draws every epoch's sample order with ``rng.permutation(m)`` on
the trainer's generator (train.py:332-347).  For a multi-million-sample pool
that is ~0.05 s of host time per epoch, more than a whole GPU step.  Here a
helper process (this file run as a script: numpy only, no torch or CUDA) keeps a copy of the generator, replays the RNG calls the trainer will
make between epoch boundaries (one ``integers(n)`` slice pick per step),
computes each permutation into a memory-mapped slot and reports the generator
state just before and just after it.  The helper runs TWO epochs ahead of the
trainer, so a permutation has a whole epoch of GPU steps to be computed in.
The trainer adopts a permutation only if its own generator state at the
boundary equals the reported pre-state, so the batch sequence is bit-identical
to drawing inline; on any mismatch (an RNG call the schedule did not predict)
it draws inline and restarts the chain, and while the helper is still starting
up it draws inline rather than wait.

Three slots rotate: the permutation in use, the next one, and the one being
computed.
"""

from __future__ import annotations

import collections
import os
import pickle
import select
import struct
import subprocess
import sys
import tempfile

import numpy as np

NSLOTS = 3


def _serve(path, m):
    slots = np.memmap(path, dtype=np.int64, mode="r+", shape=(NSLOTS, m))
    inp, out = sys.stdin.buffer, sys.stdout.buffer
    rng = None
    while True:
        try:
            msg = pickle.load(inp)
        except EOFError:
            break
        if msg is None:
            break
        kind, slot, calls = msg[0], msg[1], msg[2]
        if kind == "init":
            state = msg[3]
            rng = np.random.Generator(getattr(np.random, state["bit_generator"])())
            rng.bit_generator.state = state
        for n in calls:
            rng.integers(n)
        pre = rng.bit_generator.state
        slots[slot] = rng.permutation(m)
        msg = pickle.dumps((pre, rng.bit_generator.state))
        out.write(struct.pack("<I", len(msg)) + msg)  # length-framed: the reader never over-reads
        out.flush()


class EpochPermuter:
    """Prefetches ``rng.permutation(m)`` two epochs ahead of the trainer."""

    def __init__(self, m):
        self.m = int(m)
        d = "/dev/shm" if os.path.isdir("/dev/shm") else None
        fd, self._path = tempfile.mkstemp(prefix="mgauss_perm_", dir=d)
        os.close(fd)
        self._slots = np.memmap(self._path, dtype=np.int64, mode="w+", shape=(NSLOTS, self.m))
        # run this file as a script: numpy only (``-m package._permuter`` would
        # import the package, i.e. torch, and take seconds to start)
        self._proc = subprocess.Popen([sys.executable, os.path.abspath(__file__), self._path, str(self.m)],
                                      stdin=subprocess.PIPE, stdout=subprocess.PIPE)
        self._queue = collections.deque()  # slots of requested permutations, oldest first
        self._stale = 0  # responses still to come for abandoned requests
        self._next_slot = 0
        self._answered = False  # the helper has finished starting up (answered once)
        self._rbuf = bytearray()  # bytes read from the helper, not yet parsed
        self._fd = self._proc.stdout.fileno()
        self.adopted = 0  # epochs served from the helper

    # -- transport -----------------------------------------------------------
    def _complete(self):
        if len(self._rbuf) < 4:
            return False
        return len(self._rbuf) >= 4 + struct.unpack_from("<I", self._rbuf)[0]

    def _ready(self):
        """A whole response is available without blocking (several may be in
        flight, so bytes are buffered here rather than in a file object)."""
        while not self._complete() and select.select([self._fd], [], [], 0.0)[0]:
            data = os.read(self._fd, 1 << 16)
            if not data:
                break
            self._rbuf += data
        return self._complete()

    def _recv(self):
        while not self._complete():
            data = os.read(self._fd, 1 << 16)
            if not data:
                raise EOFError("permutation helper exited")
            self._rbuf += data
        n = struct.unpack_from("<I", self._rbuf)[0]
        out = pickle.loads(bytes(self._rbuf[4:4 + n]))
        del self._rbuf[:4 + n]
        self._answered = True
        return out

    def _send(self, msg):
        pickle.dump(msg, self._proc.stdin)
        self._proc.stdin.flush()

    def _slot(self):
        s = self._next_slot
        self._next_slot = (s + 1) % NSLOTS
        return s

    def _drain(self):
        """Drop stale responses that have arrived; True once none are left."""
        while self._stale and self._ready():
            self._recv()
            self._stale -= 1
        return self._stale == 0

    def _abandon(self):
        self._stale += len(self._queue)
        self._queue.clear()

    # -- trainer interface ---------------------------------------------------
    @property
    def chained(self):
        """Requests are outstanding (the helper's generator follows the trainer's)."""
        return bool(self._queue)

    def start(self, rng, calls_next, calls_after):
        """(Re)start the chain from rng's current state: the permutation after
        the ``integers(n)`` draws ``calls_next``, then the one after the further
        draws ``calls_after``.  Skipped while stale responses are in flight."""
        if not self._drain():
            return
        s = self._slot()
        self._send(("init", s, list(calls_next), rng.bit_generator.state))
        self._queue.append(s)
        self.extend(calls_after)

    def extend(self, calls):
        """Queue the permutation that follows the last requested one and the
        further draws ``calls``."""
        s = self._slot()
        self._send(("next", s, list(calls)))
        self._queue.append(s)

    def take(self, rng):
        """The oldest requested permutation if it was drawn from rng's current
        state (rng then advances past it), else None (the chain is dropped)."""
        if not self._queue:
            return None
        if not self._answered and not self._ready():
            # still starting up (importing numpy): draw inline rather than wait
            self._abandon()
            return None
        slot = self._queue.popleft()
        try:
            pre, post = self._recv()
        except Exception:
            self._abandon()
            return None
        if pre != rng.bit_generator.state:
            self._abandon()
            return None
        rng.bit_generator.state = post
        self.adopted += 1
        return self._slots[slot]

    def close(self):
        proc, self._proc = getattr(self, "_proc", None), None
        if proc is not None:
            try:
                pickle.dump(None, proc.stdin)
                proc.stdin.close()
                proc.wait(timeout=5)
            except Exception:
                proc.kill()
        self._slots = None
        try:
            os.unlink(self._path)
        except OSError:
            pass


if __name__ == "__main__":
    _serve(sys.argv[1], int(sys.argv[2]))
