"""Run-time variants of the S4 engine under the parity tests: the IWPP, reconstruction and
whole-pipeline parity tests of test_gpu_parity.py re-run in a subprocess with each engine
setting of k_region.cu: HP_RG_INIT (Vincent's raster / anti-raster initialisation per region
before the queue engine), HP_RG_ADI (alternating row / column phase closure of a region
instead of asynchronous sub-tile sweeps) and HP_RG_THIN (that closure only for jobs with at most
k dirty sub-tile rows; 4096 = every job), optionally only from a region's HP_RG_CHAIN-th job on."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("setting", ["HP_RG_INIT=0", "HP_RG_INIT=1", "HP_RG_ADI=0", "HP_RG_ADI=1",
                                     "HP_RG_THIN=0", "HP_RG_THIN=8", "HP_RG_THIN=4096",
                                     "HP_RG_THIN=4096,HP_RG_CHAIN=2"])
def test_s4_engine_variant(setting):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, **dict(kv.split("=") for kv in setting.split(",")))
    sel = "iwpp or recon or pipeline_config1 or pipeline_random_small or pipeline_islands or hot_path_stages_random"
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-q", "-x", "-k", sel,
                        "-p", "no:cacheprovider"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
