#!/bin/sh
# Regenerate the committed golden fixtures from the UNMODIFIED reference
# (needs /root/reference; run from the repo root). Test infrastructure only.
set -e
make -C oracle ref
oracle/_ref/fsi_ref_harness export chan tests/golden/chan.fsix --rtol 1e-8 --max-iters 300
oracle/_ref/fsi_ref_harness export chan tests/golden/chan_as.fsix --rtol 1e-8 --max-iters 300 --smoother as
oracle/_ref/fsi_ref_harness blocks tests/golden/blocks.fsix
oracle/_ref/fsi_ref_harness export cfg0 data/cfg0.fsix
oracle/_ref/fsi_ref_harness export cfg0 data/cfg0_as.fsix --smoother as
