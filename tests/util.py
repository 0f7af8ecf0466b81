import numpy as np


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def np_(t):
    return t.detach().cpu().numpy()


def gauss(m, sigma):
    j = np.arange(-m, m + 1, dtype=np.float64)
    w = np.exp(-j * j / (2 * sigma * sigma))
    return w / w.sum()


def onesided(taps, rate):
    w = np.zeros(2 * (taps - 1) + 1)
    w[taps - 1:] = np.exp(-rate * np.arange(taps))
    return w / w.sum()
