"""CPU checkers for the B200 hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and only
as the checker or the timed CPU baseline — never as the product path.

* :mod:`oracle.port`   — ctypes binding of ``liboracle.so``, the plain-C
  restatement of the reference algorithm (``splat_oracle.c``).
* :mod:`oracle.refbind` — ctypes binding of ``_ref/libsplatlm_ref.so``, the
  unmodified reference compiled from ``/root/reference/proj/src`` by
  ``oracle/Makefile`` (present wherever it was built; it travels to the GPU
  box with the snapshot, but ``/root/reference`` itself does not).
"""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsplatlm_ref.so")
PORT_SO = os.path.join(HERE, "liboracle.so")


def build(ref: bool = True) -> None:
    """Build the C restatement and, when /root/reference is present, the reference."""
    target = ["all"] if ref else ["oracle"]
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *target], check=True)


def have_ref() -> bool:
    return os.path.exists(REF_SO)
