"""Restatement of scikit-image's published structural_similarity (>=0.21).

Pinned contract (reference pyproject pins ``scikit-image>=0.21``, no lockfile):
gaussian weights, sigma=1.5, truncate=3.5 -> 11x11 window, ``mode='reflect'``
scipy filtering, population covariance when use_sample_covariance=False,
C1=(0.01 R)^2, C2=(0.03 R)^2, S-map cropped by (win-1)/2 on every side and
averaged in float64; multichannel images are scored per channel and averaged.
Test infrastructure only (fixture generation); never imported by the product.
"""
import numpy as np
from scipy.ndimage import gaussian_filter


def structural_similarity(im1, im2, *, win_size=None, gradient=False, data_range=None,
                          channel_axis=None, gaussian_weights=False, full=False, **kwargs):
    if gradient or full:
        raise NotImplementedError("shim supports the mean-SSIM path only")
    im1 = np.asarray(im1, dtype=np.float64)
    im2 = np.asarray(im2, dtype=np.float64)
    if im1.shape != im2.shape:
        raise ValueError("Input images must have the same dimensions.")
    if channel_axis is not None:
        nch = im1.shape[channel_axis]
        vals = [structural_similarity(np.take(im1, c, axis=channel_axis),
                                      np.take(im2, c, axis=channel_axis),
                                      win_size=win_size, data_range=data_range,
                                      gaussian_weights=gaussian_weights, **kwargs)
                for c in range(nch)]
        return float(np.mean(vals))
    K1 = kwargs.pop("K1", 0.01)
    K2 = kwargs.pop("K2", 0.03)
    sigma = kwargs.pop("sigma", 1.5)
    use_sample_covariance = kwargs.pop("use_sample_covariance", True)
    if not gaussian_weights:
        raise NotImplementedError("shim supports gaussian_weights=True only")
    truncate = 3.5
    if win_size is None:
        win_size = 2 * int(truncate * sigma + 0.5) + 1
    if any(s < win_size for s in im1.shape):
        raise ValueError("win_size exceeds image extent")
    if data_range is None:
        raise ValueError("data_range required in shim")

    def filt(x):
        return gaussian_filter(x, sigma=sigma, mode="reflect", truncate=truncate)

    ndim = im1.ndim
    NP = win_size ** ndim
    cov_norm = NP / (NP - 1) if use_sample_covariance else 1.0
    ux, uy = filt(im1), filt(im2)
    uxx, uyy, uxy = filt(im1 * im1), filt(im2 * im2), filt(im1 * im2)
    vx = cov_norm * (uxx - ux * ux)
    vy = cov_norm * (uyy - uy * uy)
    vxy = cov_norm * (uxy - ux * uy)
    R = data_range
    C1 = (K1 * R) ** 2
    C2 = (K2 * R) ** 2
    A1, A2, B1, B2 = (2 * ux * uy + C1, 2 * vxy + C2, ux ** 2 + uy ** 2 + C1, vx + vy + C2)
    S = (A1 * A2) / (B1 * B2)
    pad = (win_size - 1) // 2
    sl = tuple(slice(pad, s - pad) for s in S.shape)
    return float(S[sl].mean(dtype=np.float64))
