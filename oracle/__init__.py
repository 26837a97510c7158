"""ORACLE — test infrastructure only.

CPU restatement (numpy, f64) of the reference's hot path, used as the checker by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg — never by the product path
(paper_2310_16355_b200 does not import this package).

  rng_ref.py    RngStream (rng.hpp:15-91) and init_transformer_params (model.hpp:49-70)
  model_ref.py  transformer_logits / transformer_loss forward (model.hpp:76-152) and the
                reverse-mode gradients autodiff.hpp would emit, AdamW (train_state.hpp:183-220),
                the audit trajectory (audit.hpp:78-159)
  _ref/         the reference itself, compiled from /root/reference by oracle/Makefile

Parity of this restatement is pinned against the reference's own outputs
(tests/golden/*.npz, produced by oracle/_ref/sw_ref_driver) in tests/test_oracle.py.
"""
