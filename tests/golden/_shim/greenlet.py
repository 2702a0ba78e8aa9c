"""Minimal thread-backed stand-in for the `greenlet` package.

Test infrastructure only: the reference's simulated transport
(/root/reference/pkg/src/minidist/transport/sim.py:25) imports greenlet at
module top, and greenlet has no offline wheel in this image. The reference
uses exactly three operations -- ``greenlet(run)``, ``getcurrent()`` and
``g.switch()`` -- with one scheduler greenlet handing control to rank
greenlets and each rank switching back (sim.py:105, :360, :390-393). This
shim runs every greenlet on its own OS thread and lets exactly one of them
hold a baton at a time, which reproduces those semantics (including "a
finished greenlet returns control to its parent").
"""

import threading

_local = threading.local()


class greenlet:  # noqa: N801 - mirrors the real package's class name
    def __init__(self, run=None, parent=None):
        self._run = run
        self.parent = parent if parent is not None else getcurrent()
        self._go = threading.Semaphore(0)
        self._thread = None
        self.dead = False
        self._value = None

    def _bootstrap(self):
        _local.current = self
        self._go.acquire()
        try:
            self._run()
        finally:
            self.dead = True
            self.parent._value = None
            self.parent._go.release()

    def switch(self, *args):
        me = getcurrent()
        if self is me:
            return None
        if self._thread is None and self._run is not None:
            self._thread = threading.Thread(target=self._bootstrap, daemon=True)
            self._thread.start()
        self._go.release()
        me._go.acquire()
        return me._value


class _Root(greenlet):
    def __init__(self):
        self._run = None
        self.parent = None
        self._go = threading.Semaphore(0)
        self._thread = threading.current_thread()
        self.dead = False
        self._value = None


def getcurrent():
    cur = getattr(_local, "current", None)
    if cur is None:
        cur = _Root()
        _local.current = cur
    return cur
