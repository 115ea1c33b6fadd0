"""ORACLE — test infrastructure, never product code.

A CPU float64 restatement of the reference's (`splatstream`, /root/reference)
sliding-window training hot path, used only as

* the parity checker for the CUDA path (``tests/``, ``__graft_entry__.smoke``),
* the CPU baseline timed by ``bench.py`` (``cpu_baseline`` and
  ``--impl reference``).

Every function cites the reference file:line it restates.  The restatement
is pinned against golden vectors produced by the reference itself
(``tests/golden/make_golden.py`` imports the reference in the build
container and writes ``tests/golden/*.npz``; ``tests/test_oracle_golden.py``
checks this package against them).

The product package (``paper_2409_07759_b200``) must never import this
package.
"""
