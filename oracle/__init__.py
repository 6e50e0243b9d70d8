"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference `isingsynth` generation loop
(/root/reference/pkg/src/isingsynth: engine.py, ga.py, encoding.py, gates.py,
fitness.py) with the reference's sequential numpy Generators replaced by the
counter-based Philox stream scheme the device uses (oracle/streams.py,
paper_1809_11134_b200/csrc/np_random.cuh).  Every function cites the reference
file:line it restates.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import
this package, and only as the checker / the timed CPU reference; the product
package (paper_1809_11134_b200) never imports it.

Pinning: oracle/gen_golden.py drives the reference's OWN functions (imported
from /root/reference in the build container) with the same per-unit Philox
generators and commits the outputs as tests/golden/*.npz; tests/test_oracle.py
checks this restatement against those fixtures and against the reference's own
known-answer values.
"""
