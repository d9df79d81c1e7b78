"""Grid operations (reference ``gridops.py``), numpy in / numpy out."""

from paper_1807_05117_b200 import gridops as _g

from ._conv import dev, host


def warp(domain, values, displacement, interp="linear"):
    return host(_g.warp(domain, dev(domain, values, False), dev(domain, displacement, False), interp))


def fourier_warp(domain, values, displacement):
    return host(_g.fourier_warp(domain, dev(domain, values, False), dev(domain, displacement, False)))


def spatial_gradient(domain, values, mode="central"):
    return host(_g.spatial_gradient(domain, dev(domain, values, False), mode))


def jacobian_matrix(domain, displacement):
    return host(_g.jacobian_matrix(domain, dev(domain, displacement, False)))


def jacobian_determinant(domain, displacement):
    return host(_g.jacobian_determinant(domain, dev(domain, displacement, False)))
