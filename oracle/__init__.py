"""SAGIPS oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, single-threaded-in-spirit CPU implementation (numpy, float64)
of the per-rank GAN training step of SAGIPS (arXiv 2407.00051) and of its
ring exchange of generator weight gradients, written directly from the paper
(PAPER.md, cited as P:<line>) and from the readings recorded in DESIGN.md
("Readings" table, cited as R<n>).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2407_00051_b200``) never imports it and shares no code
with it: the Philox generator, the sampler, the MLPs, the loss, Adam and the
exchange are all written a second time here, independently of the CUDA
sources.

Modules
  philox    -- Philox4x32-10 counter-based RNG, uniform and Box-Muller maps
  proxy     -- the proxy pipeline f(x_hat(p)) (Eq. 4/5):
               constrain, inverse-CDF quantile sampler, reference data,
               50% bootstrap shard, bootstrap batch, histograms, and the
               sampler backward (dL/dc)
  mlp       -- MLP forward/backward, LeakyReLU, BCE-with-logits, Adam,
               Kaiming-normal init
  exchange  -- group layout, Alg. 1 ring all-reduce read as a
               pass-along ring with an ascending fold (R10),
               outer leaders' ring every h steps, modes (Tab. III)
  gan       -- the whole per-rank step and a lockstep
               multi-rank driver
  ensemble  -- ensemble response (Eq. 7/8), normalised residuals (Eq. 6)
               and the split-batch rule (Eq. 10)
  tabulated -- the tabulated-CDF sampler variant:
               density on a grid, trapezoid CDF, binary-search inversion,
               exact backward of the tabulated inverse

Every function here is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` against something other than itself (published
known-answer vectors, closed forms, brute force, finite differences); the
training trajectories (N=1 and multi-rank, every exchange mode) are pinned
against the same loop written with PyTorch autograd + torch.optim.Adam.
"""
