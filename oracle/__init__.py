"""ORACLE -- test infrastructure, not product code.

A CPU restatement of the reference's (``nysode``, /root/reference/pkg/src) hot
path in NumPy: ``nys_port`` (kernel, Nystrom feature map, linear KKT) and
``newton_port`` (Newton-KKT ladder).  Pinned against golden vectors produced by
the live reference (``tests/golden/make_golden.py``).

Import rule: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and only
as the checker or the timed CPU baseline.  The product package
``paper_2510_04094_b200`` never imports it and has no CPU fallback.
"""
