"""paper_1808_00685_b200 -- B200-native generalised 2D correlation (corr2D).

Drop-in for the reference package ``corrtwo`` 0.1.0's Fourier-route hot path
(preprocess_dataset -> dft_channels -> correlate_ft), plus the Hilbert route
(correlate_ht): same names, arguments,
defaults, result layout and error classes, executed by hand-written sm_100a
CUDA kernels (libcorr2d.so, C ABI in include/corr2d.h).  There is no CPU
fallback: without the built library or a CUDA device every compute entry
point raises ``BackendUnavailable``.
"""

__version__ = "0.1.0"

from ._abi import BackendUnavailable
from .analysis import (AutoPeak, CrossPeak, CrossPeakVerdict, PeakReport, Verdict, classify_cross_peak,
                       find_peaks)
from .api import corr2d
from .dataset import CorrelationSpectra, SpectralDataset
from .engine_core import NormalizationSpec, check_pair, is_same_dynamic, row_blocks
from .errors import CorrtwoError, DataError, NumericError, ParseError
from .fourier import (DeviceCorrelationSpectra, FourierWorkspace, correlate_ft, dft_channels,
                      half_spectrum_weights)
from .hilbert import correlate_ht, hilbert_noda_matrix, hilbert_transform, sync_direct
from .serialize import (LONG_FORM, MATRIX_PAIR, correlation_paths, format_number, save_correlation,
                        write_correlation)
from .preprocess import (DynamicSpectra, InterpolantKind, PreprocessSpec, ReferenceSpec,
                         ResampleSpec, apply_scaling, default_target_count, dynamic_spectra,
                         mean_reference, preprocess_dataset, resample_equidistant,
                         resample_to_axis, stddev_spectrum)

__all__ = [
    "AutoPeak", "BackendUnavailable", "CorrelationSpectra", "CrossPeak", "CrossPeakVerdict", "PeakReport",
    "Verdict", "classify_cross_peak", "find_peaks", "CorrtwoError", "DataError", "DeviceCorrelationSpectra",
    "DynamicSpectra", "FourierWorkspace", "InterpolantKind", "NormalizationSpec", "NumericError",
    "ParseError", "PreprocessSpec", "ReferenceSpec", "ResampleSpec", "SpectralDataset",
    "apply_scaling", "check_pair", "correlate_ft", "correlate_ht", "corr2d", "default_target_count",
    "dft_channels", "dynamic_spectra", "half_spectrum_weights", "hilbert_noda_matrix",
    "hilbert_transform", "is_same_dynamic",
    "mean_reference", "preprocess_dataset", "resample_equidistant", "resample_to_axis",
    "row_blocks", "stddev_spectrum", "sync_direct", "LONG_FORM", "MATRIX_PAIR", "correlation_paths",
    "format_number", "save_correlation", "write_correlation",
]
