"""A checkpoint blob written by the REFERENCE package's codec
(fedsim.fault.save_checkpoint, pkg/src/fedsim/fault.py:147-172), for the
byte-compatibility test of the framework's codec.

Usage:  oracle/build_ref.sh && python tests/golden/make_golden_ckpt.py
Writes tests/golden/ckpt_ref.bin.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))


def main() -> None:
    from oracle.ref_pool import use_reference

    use_reference("compiled")
    from fedsim.fault import Checkpoint, save_checkpoint
    from fedsim.model import ParamVector

    values = np.linspace(-1.5, 2.5, 97) ** 3
    ck = Checkpoint(scope="client-7", round=3, seq=11, params=ParamVector(values, "abcdef0123456789"),
                    optimizer_state={"lr": 0.05, "train_seed": 12345}, epoch=2, batch_index=5)
    with open(os.path.join(HERE, "ckpt_ref.bin"), "wb") as f:
        f.write(save_checkpoint(ck))


if __name__ == "__main__":
    main()
