"""A short run of the randomised parity campaign (tests/fuzz_parity.py): random
inputs and random kernel-choice knobs, every result bit for bit against the
compiled reference. Longer campaigns: `python tests/fuzz_parity.py --seconds N`."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [20260115, 458])
def test_fuzz_campaign(ref, seed):
    from fuzz_parity import Campaign

    counts, failures = Campaign(seed).run(seconds=20, max_cases=140)
    assert not failures, failures[:3]
    assert sum(counts.values()) >= 7
