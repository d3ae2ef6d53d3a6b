"""Host-side pins of bench.py's measurement model (no GPU): the per-kernel flop counts are
checked against explicit operation counts of the loops they model, and the kernel-choice
mirror against the launcher's rule (csrc/demod_inst.cu launch_strip, csrc/demod_strip.cuh
strip_kind)."""

import pytest

import bench


def _count_covariance_full(M):
    # R_ij += a_i·conj(a_j) for j < i (one complex MAC = 8 flops) and the real diagonal
    # |a_i|² (2 FMAs = 4 flops), for each of the M window columns
    return M * (M * (M - 1) // 2 * 8 + M * 4)


def _count_new_row(M):
    # the new last row only: M−1 complex MACs and one diagonal entry per column
    return M * ((M - 1) * 8 + 4)


@pytest.mark.parametrize("M", [3, 8, 11, 16, 32])
def test_covariance_counts(M):
    full = _count_covariance_full(M)
    # the model's 4M³ is the leading term of the explicit count (it omits the −4M² + 4M part)
    assert abs(bench.covariance_flops(M, None) - full) <= 4 * M * M
    for S in (1, 2, 16):
        expect = (4.0 * M ** 3 + (S - 1) * _count_new_row(M)) / S
        assert bench.covariance_flops(M, S) == pytest.approx(expect)


def test_implicit_kernel_has_no_covariance_and_doubles_the_matvec():
    M, k = 20, 3.0
    explicit = bench.flops_per_pixel(M, k, 1.0, 1.0, strip_rows=None)
    implicit = bench.flops_per_pixel(M, k, 1.0, 1.0, kind=2)
    # implicit − explicit = 12M² + k·8M² − 4M³ (one window pass, the second matvec, no build)
    assert implicit - explicit == pytest.approx(12 * M * M + k * 8 * M * M - 4 * M ** 3)


def test_strip_kind_and_rows_mirror_the_launcher():
    assert [bench.strip_kind(M) for M in (3, 8, 10, 11, 12, 13, 14, 20, 32)] == [1, 1, 1, 2, 1, 1, 2, 2, 2]
    # the bench stack (99 flow frames of 1024²) runs 16-row strips at every M
    assert all(bench.strip_rows_for(M, 99, 1024, 1024) == 16 for M in range(3, 33))
    # one 512² frame is too small for 8-row strips: the row kernel runs it
    assert bench.strip_rows_for(8, 1, 512, 512) is None
    assert bench.kernel_name(8, 1, 512, 512).startswith("bos::demod_kernel<8")
    assert bench.kernel_name(20, 1, 512, 512) == "bos::demod_strip_im_kernel<20,false>"   # any size from M = 17
    assert bench.kernel_name(8) == "bos::demod_strip_kernel<8,false>"
    assert bench.kernel_name(20) == "bos::demod_strip_im_kernel<20,false>"
