"""Helpers for the -m gpu parity tests: numpy <-> column-major CUDA tensors."""
import numpy as np


def to_dev(M):
    import torch
    from paper_2602_19090_b200 import colmajor
    return colmajor(torch.from_numpy(np.ascontiguousarray(M, dtype=np.float64)).cuda())


def to_np(T):
    return T.detach().cpu().numpy()


def vec_dev(v):
    import torch
    return torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).cuda()
