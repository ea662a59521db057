"""Q-Palette CPU oracle (NumPy, float64) -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import anything under `oracle/`. The CUDA product
path (`paper_2509_20214_b200`) never imports it, and the two share no code: the
oracle implements the paper's definitions directly, slowly and in float64, so a
reader can check each function against the cited passage of
/root/reference/PAPER.md ("P:n" = line n).

Modules
  codebooks  NUQ (Lloyd-Max), uniform SQ, 2-D VQ (k-means), TCQ tlut + quantlut_sym
  rht        randomized Hadamard rotation R = (1/sqrt(b)) blockdiag(H_b) D
  layout     the frozen code layout of LAYOUT.md (tile / lane / step -> weights)
  decode     dq(r; LUT) for TCQ, half-TCQ, VQ, NUQ, UNIF
  encode     RTN and tail-biting Viterbi
  linear     y = diag(s) W_hat R x and the data-free offline path
  allocation Theorem 1 optimal fractional bit allocation
  msq        fusion-aware mixed-scheme quantization by brute force (tiny instances)

Parity status of every function is listed in DESIGN.md ("Oracle pins");
functions without an external pin say "parity unpinned" in their docstring.
"""
