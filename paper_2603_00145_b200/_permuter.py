"""Epoch permutations computed ahead in a helper process.

The reference draws every epoch's sample order with ``rng.permutation(m)`` on
the trainer's generator (train.py:332-347).  For a multi-million-sample pool
that is ~0.1 s of host time per epoch, more than a whole GPU step.  Here a
helper process (``python -m paper_2603_00145_b200._permuter``: numpy only, no
CUDA) takes a copy of the generator state, replays the RNG calls the trainer
will make before its next epoch boundary, computes the permutation into a
memory-mapped buffer and reports the generator state just before and just
after it.  The trainer adopts the result only if its own state at the boundary
equals the reported pre-state, so the batch sequence is bit-identical to
drawing the permutation inline; on any mismatch, or when the result is not
ready at the boundary (the trainer never waits for the helper), it draws
inline.

Two buffer slots alternate: the permutation in use stays valid while the
helper fills the other one.
"""

from __future__ import annotations

import os
import pickle
import select
import subprocess
import sys
import tempfile

import numpy as np


def _serve(path, m):
    slots = np.memmap(path, dtype=np.int64, mode="r+", shape=(2, m))
    inp, out = sys.stdin.buffer, sys.stdout.buffer
    while True:
        try:
            msg = pickle.load(inp)
        except EOFError:
            break
        if msg is None:
            break
        slot, state, calls = msg
        rng = np.random.Generator(getattr(np.random, state["bit_generator"])())
        rng.bit_generator.state = state
        for n in calls:
            rng.integers(n)
        pre = rng.bit_generator.state
        slots[slot] = rng.permutation(m)
        pickle.dump((pre, rng.bit_generator.state), out)
        out.flush()


class EpochPermuter:
    """Prefetches ``rng.permutation(m)`` for the trainer's next epoch."""

    def __init__(self, m):
        self.m = int(m)
        d = "/dev/shm" if os.path.isdir("/dev/shm") else None
        fd, self._path = tempfile.mkstemp(prefix="mgauss_perm_", dir=d)
        os.close(fd)
        self._slots = np.memmap(self._path, dtype=np.int64, mode="w+", shape=(2, self.m))
        env = dict(os.environ)
        pkg_parent = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        env["PYTHONPATH"] = pkg_parent + (os.pathsep + env["PYTHONPATH"] if env.get("PYTHONPATH") else "")
        self._proc = subprocess.Popen([sys.executable, "-m", "paper_2603_00145_b200._permuter", self._path,
                                       str(self.m)], stdin=subprocess.PIPE, stdout=subprocess.PIPE, env=env)
        self._pending = None  # slot being filled
        self._stale = False  # a result nobody will take is still on its way
        self._slot = 0
        self.adopted = 0  # epochs served from the helper

    def _recv(self):
        return pickle.load(self._proc.stdout)

    def _ready(self):
        """A response can be read without blocking (at most one is ever in
        flight, so nothing is left in the reader's buffer between responses)."""
        return bool(select.select([self._proc.stdout], [], [], 0.0)[0])

    def request(self, rng, integer_calls):
        """Start computing the permutation that follows the given further
        ``rng.integers(n)`` draws (one n per call) from rng's current state.
        Skipped (the trainer then draws that epoch inline) while the helper is
        still busy with an earlier request."""
        if self._pending is not None or self._stale:
            if not self._ready():
                return
            self._recv()  # drop the stale result
            self._pending, self._stale = None, False
        self._slot ^= 1
        self._pending = self._slot
        pickle.dump((self._slot, rng.bit_generator.state, list(integer_calls)), self._proc.stdin)
        self._proc.stdin.flush()

    def take(self, rng):
        """The prefetched permutation if it was drawn from rng's current
        state (rng then advances past it), else None."""
        if self._pending is None:
            return None
        slot, self._pending = self._pending, None
        if not self._ready():  # not done yet (e.g. the helper is still starting): draw inline
            self._stale = True
            return None
        try:
            pre, post = self._recv()
        except Exception:
            return None
        if pre != rng.bit_generator.state:
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
