import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libfsb_b200.so")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN, "golden.npz"))


@pytest.fixture(scope="session")
def digests():
    import json

    with open(os.path.join(GOLDEN, "digests.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def full_models():
    from paper_2603_15603_b200 import synth

    return synth.make_toy_models(0, 18439, 6890)


@pytest.fixture(scope="session")
def toy_models():
    from paper_2603_15603_b200 import synth

    return synth.make_toy_models(0, 1200, 600)


@pytest.fixture(scope="session")
def dec_weights():
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import synth

    return synth.decoder_weights(dc.DecoderConfig(), 40)


def projector_dict(pw):
    return dict(w1=pw.w1, b1=pw.b1, w2=pw.w2, b2=pw.b2, w3=pw.w3, b3=pw.b3, subsample=pw.subsample, mask=pw.mask)


@pytest.fixture(scope="session")
def full_projector():
    from paper_2603_15603_b200 import projection as pj

    return pj.init_projector(pj.make_subsample(6890, 1500), (512, 256), seed=0)


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = max(np.abs(b).max(), 1e-30)
    return float(np.abs(a - b).max() / den)
