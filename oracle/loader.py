"""Parallel loading process (Algorithm 1): the preprocessing
and the sequence of batches the trainer receives.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Alg. 1: load the batch file into hostdata_x, subtract the mean image,
crop and mirror according to the mode, transfer to the GPU.  The paper leaves
the crop geometry and the mirror rule open (reading Q20 in
DESIGN.md): TRAIN takes, for example b of the f-th file loaded,
    z = splitmix64(seed ^ splitmix64((f << 32) | b))
    oy = z % (h - ch + 1),  ox = (z >> 20) % (w - cw + 1),  mirror = (z >> 40) & 1
VAL takes the centre crop without mirroring.  Per element (one fp32 rounding):
    out[b, k, y, x] = fl(float(raw[b, k, oy+y, ox+xs]) - mean[k, oy+y, ox+xs]),
    xs = cw - 1 - x if mirror else x.

deliveries() replays the Alg. 1 state machine over a message list and returns
which (file, mode, load index) each trainer wait() receives.

Parity status: splitmix64 pinned by published reference outputs (Vigna's
splitmix64 with seed 0 / 1234567, tests/golden/splitmix64.txt); preprocess
pinned by SPEC L412-413 (mean == data -> zeros; VAL deterministic), an
element-by-element Python loop, crop bounds and mirror involution;
deliveries() pinned by hand-derived sequences for the cases of SPEC L420-422.
"""

import struct

import numpy as np

MASK = (1 << 64) - 1


def splitmix64(z):
    """Vigna's SplitMix64 output function (one step from state z)."""
    z = (z + 0x9E3779B97F4A7C15) & MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def crop_params(n, h, w, ch, cw, mode, seed, file_index):
    """[(oy, ox, mirror)] for the n examples of the file_index-th loaded file."""
    out = []
    for b in range(n):
        if mode == "train":
            z = splitmix64((seed ^ splitmix64(((file_index << 32) | b) & MASK)) & MASK)
            out.append((z % (h - ch + 1), (z >> 20) % (w - cw + 1), (z >> 40) & 1))
        else:
            out.append(((h - ch) // 2, (w - cw) // 2, 0))
    return out


def preprocess(raw, mean, ch, cw, mode, seed, file_index):
    """raw: uint8 [n, c, h, w]; mean: float32 [c, h, w].  Mean subtraction on the
    full image first (Alg. 1), then crop and mirror (L341)."""
    n, c, h, w = raw.shape
    centred = np.subtract(raw.astype(np.float32), mean[None].astype(np.float32), dtype=np.float32)
    out = np.empty((n, c, ch, cw), np.float32)
    for b, (oy, ox, mir) in enumerate(crop_params(n, h, w, ch, cw, mode, seed, file_index)):
        win = centred[b, :, oy:oy + ch, ox:ox + cw]
        out[b] = win[:, :, ::-1] if mir else win
    return out


def read_batch_file(path):
    """"PXB1" | u32 n, c, h, w (little endian) | n*c*h*w uint8 (NCHW)."""
    with open(path, "rb") as f:
        head = f.read(20)
        if len(head) != 20 or head[:4] != b"PXB1":
            raise ValueError("not a PXB1 batch file")
        n, c, h, w = struct.unpack("<4I", head[4:])
        data = np.frombuffer(f.read(), dtype=np.uint8)
    if data.size != n * c * h * w:
        raise ValueError("truncated payload")
    return data.reshape(n, c, h, w)


def deliveries(messages):
    """Replay Alg. 1 over trainer messages [("train"|"val"|"stop"|"file", name)].
    Returns [(file, mode, load_index)] in the order the trainer receives them;
    load_index counts every file loaded (delivered or not)."""
    out, i, loads = [], 0, 0
    msg = messages[i] if i < len(messages) else ("stop", None)
    i += 1
    while True:
        if msg[0] == "stop":
            return out
        mode = msg[0]
        msg = messages[i] if i < len(messages) else ("stop", None)
        i += 1
        if msg[0] != "file":
            return out
        current = (msg[1], mode, loads)
        while True:
            loads += 1                      # L339-342: load + preprocess `current`
            msg = messages[i] if i < len(messages) else ("stop", None)
            i += 1                          # L343
            if msg[0] != "file":
                break                       # L344-345: msg is the next mode
            out.append(current)             # L350-352: deliver the loaded batch
            current = (msg[1], mode, loads)
