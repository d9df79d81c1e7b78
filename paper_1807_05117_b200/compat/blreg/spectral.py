"""Spectral algebra (reference ``spectral.py``), numpy in / numpy out; the
transforms, truncated convolutions and diagonal operators run on the device."""

import numpy as np

from paper_1807_05117_b200 import spectral as _s

from ._conv import dev, host


def conjugate_reverse(coeffs, ndim):  # spectral.py:37-42
    out = np.asarray(coeffs)
    for ax in range(-ndim, 0):
        out = np.roll(np.flip(out, axis=ax), 1, axis=ax)
    return np.conj(out)


def symmetrize(coeffs, ndim):  # spectral.py:45-47
    return 0.5 * (np.asarray(coeffs) + conjugate_reverse(coeffs, ndim))


def symmetry_error(coeffs, ndim):  # spectral.py:50-56
    c = np.asarray(coeffs)
    scale = float(np.max(np.abs(c))) if c.size else 0.0
    if scale == 0.0:
        return 0.0
    return float(np.max(np.abs(c - conjugate_reverse(c, ndim)))) / scale


def include(domain, coeffs, grid_shape=None, check=True):
    return host(_s.include(domain, dev(domain, coeffs, True), grid_shape, check=check))


def project(domain, values, grid_shape=None):
    return host(_s.project(domain, dev(domain, values, False), grid_shape))


def truncated_convolution(domain, a, b):
    return host(_s.truncated_convolution(domain, dev(domain, a, True), dev(domain, b, True)))


def conv_scalar(domain, a, b):
    return host(_s.conv_scalar(domain, dev(domain, a, True), dev(domain, b, True)))


def conv_dot(domain, a, b):
    return host(_s.conv_dot(domain, dev(domain, a, True), dev(domain, b, True)))


def conv_matvec(domain, mat, vec, transpose=False):
    return host(_s.conv_matvec(domain, dev(domain, mat, True), dev(domain, vec, True), transpose))


def metric_symbol(domain):
    return _s.metric_symbol(domain)


def apply_helmholtz(domain, coeffs):
    return host(_s.apply_helmholtz(domain, dev(domain, coeffs, True)))


def apply_inverse_helmholtz(domain, coeffs):
    return host(_s.apply_inverse_helmholtz(domain, dev(domain, coeffs, True)))


def spectral_gradient(domain, scalar):
    return host(_s.spectral_gradient(domain, dev(domain, scalar, True)))


def spectral_divergence(domain, vec):
    return host(_s.spectral_divergence(domain, dev(domain, vec, True)))


def spectral_jacobian(domain, vec):
    return host(_s.spectral_jacobian(domain, dev(domain, vec, True)))


def leray_projection(domain, vec):
    return host(_s.leray_projection(domain, dev(domain, vec, True)))


def make_divergence_free(domain, vec):
    return host(_s.make_divergence_free(domain, dev(domain, vec, True)))


def inner(a, b):  # spectral.py:335-337
    return float(np.real(np.vdot(np.asarray(b), np.asarray(a))))


def grid_inner(domain, f, g):
    return _s.grid_inner(domain, dev(domain, f, False), dev(domain, g, False))


def grid_norm2(domain, f):
    return _s.grid_norm2(domain, dev(domain, f, False))


def max_abs(domain, coeffs):
    return _s.max_abs(domain, dev(domain, coeffs, True))
