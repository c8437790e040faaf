"""The bit-exactness tests of test_gpu_dock.py re-run with the context in
MDR_PAIR_FP64 (the reference's exact double operation order, IEEE
divisions); test_gpu_dock.py itself runs the default MDR_PAIR_FP64_FAST."""
import pytest

import test_gpu_dock as T  # noqa: E402 (pytest puts tests/ on sys.path)

pytestmark = pytest.mark.gpu


def test_score_golden_fixtures_ref64(dev_ref, instances, ref_vectors):
    T.test_score_golden_fixtures(dev_ref, instances, ref_vectors)


@pytest.mark.parametrize("partition", [32, 64, 128])
def test_score_baseline_bit_exact_random_ref64(dev_ref, port, partition):
    T.test_score_baseline_bit_exact_random(dev_ref, port, partition)


def test_score_tcu_reference_compatible_ref64(dev_ref, port):
    T.test_score_tcu_reference_compatible(dev_ref, port)


def test_local_search_golden_ref64(dev_ref, instances, ref_vectors):
    T.test_local_search_golden(dev_ref, instances, ref_vectors)


def test_local_search_batch_vs_oracle_ref64(dev_ref, port, instances):
    T.test_local_search_batch_vs_oracle(dev_ref, port, instances)


def test_lga_golden_and_determinism_ref64(dev_ref, instances, ref_vectors):
    T.test_lga_golden_and_determinism(dev_ref, instances, ref_vectors)


@pytest.mark.parametrize("name", ["s1", "s3"])
def test_lga_paired_statistical_parity_ref64(dev_ref, port, instances, name):
    T.test_lga_paired_statistical_parity(dev_ref, port, instances, name)
