"""Pins for the sk-means oracle (``oracle/skmeans.py``; §4.2,
SPEC.md:92-97 and 353-360) against worked examples, closed forms and a direct cosine oracle."""
import numpy as np
import pytest

import oracle


def test_normalize_examples():
    """(3,4) -> (0.6,0.8); an exactly unit row is unchanged."""
    out = oracle.normalize_rows(np.array([[3, 4], [0, -1], [1, 0]], np.float32))
    assert out.tolist() == np.array([[0.6, 0.8], [0, -1], [1, 0]], np.float32).tolist()


def test_normalize_zero_row_is_domain_error():
    """zero row -> domain error."""
    with pytest.raises(ValueError):
        oracle.normalize_rows(np.array([[1, 2], [0, 0]], np.float32))


def test_unit_sphere_identity():
    """SPEC.md:97 / the identity that licenses MTI for sk-means: ||u-w||^2 = 2 (1 - u.w)."""
    rng = np.random.default_rng(3)
    U = oracle.normalize_rows(rng.normal(size=(200, 7)).astype(np.float32)).astype(np.float64)
    W = oracle.normalize_rows(rng.normal(size=(200, 7)).astype(np.float32)).astype(np.float64)
    lhs = ((U - W) ** 2).sum(1)
    rhs = 2.0 * (1.0 - (U * W).sum(1) / (np.linalg.norm(U, axis=1) * np.linalg.norm(W, axis=1)))
    assert np.allclose(lhs, rhs, rtol=0, atol=1e-6)   # fp32 rows are unit to ~1e-7


def test_skmeans_two_axes():
    """points (2,0),(0,3), k=2 -> normalized centroids (1,0),(0,1)."""
    r = oracle.skmeans(np.array([[2, 0], [0, 3]], np.float32), np.array([[2, 0], [0, 3]], float), 10)
    assert r.C.tolist() == [[1.0, 0.0], [0.0, 1.0]]
    assert r.a.tolist() == [0, 1] and r.iterations == 2 and r.changed.tolist() == [2, 0]


def test_skmeans_one_ray():
    """all points on one ray, k=1 -> the centroid is the ray's unit vector."""
    X = np.array([[1, 2], [2, 4], [3, 6], [0.5, 1]], np.float32)
    r = oracle.skmeans(X, X[:1].astype(float), 5)
    u = np.array([1.0, 2.0]) / np.sqrt(5.0)
    assert np.allclose(r.C[0], u, rtol=0, atol=1e-7) and r.iterations == 2


def test_skmeans_assignment_is_cosine_argmax():
    """one assignment step equals the exhaustive cosine argmax on the raw data."""
    rng = np.random.default_rng(5)
    X = rng.normal(size=(3000, 6)).astype(np.float32)
    C0 = rng.normal(size=(9, 6))
    r = oracle.skmeans(X, C0, 1)
    X64 = X.astype(np.float64)
    cos = (X64 @ C0.T) / (np.linalg.norm(X64, axis=1)[:, None] * np.linalg.norm(C0, axis=1)[None, :])
    best = np.sort(cos, axis=1)
    clear = best[:, -1] - best[:, -2] > 1e-9
    assert clear.mean() > 0.99
    assert np.array_equal(r.a[clear], cos.argmax(1)[clear])


def test_skmeans_centroids_unit_and_sse_nonincreasing():
    """Every non-empty centroid is a unit vector; SSE on the sphere does not increase."""
    rng = np.random.default_rng(9)
    X = rng.normal(size=(5000, 5)).astype(np.float32) + np.array([3, 0, 0, 0, 0], np.float32)
    r = oracle.skmeans(X, X[:7].astype(float), 30)
    assert np.allclose(np.linalg.norm(r.C, axis=1), 1.0, rtol=0, atol=1e-12)
    assert np.all(np.diff(r.sse) <= 1e-9 * r.sse[0])
