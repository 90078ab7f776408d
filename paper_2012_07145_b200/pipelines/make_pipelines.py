"""Author the BASELINE.json workload pipelines in the reference text format
(reference pkg/src/gpusched/pipeline.py:253-359; producer and consumer
ranks must match, pipeline.py:145-147).  The reference ships only blur,
conv and stencil_chain, so these are built here (SURVEY §7 hard part 7):

  unsharp          C2: 3-channel unsharp mask, 1536x2560 (8 funcs)
  harris           C2: Harris corner response, 1536x2560 (13 funcs)
  resnet_block     C4: ResNet-50 bottleneck block 56x56x256 -> 64 -> 64 -> 256
                       + skip (channel reductions as stride-0 windows, as the
                       reference's conv.txt does)
  resnet_small     the same block at 28x28x32 -> 8 -> 8 -> 32, small enough
                       for the reference's brute-force featurizer (goldens)
  camera_pipe      C3: ~100-func camera pipeline (hot-pixel suppression,
                       Bayer deinterleave by stride-2 reads, demosaic,
                       colour matrix, tone curve, sharpening)
  local_laplacian  C3: ~100-func local Laplacian filter (Gaussian / Laplacian
                       pyramids with stride-2 downsampling)

Integer strides cannot express upsampling (x/2, pipeline.py:27-30), so the
pyramid's upsample steps ("expand" funcs at the fine size) read the coarse
level at stride 1 with a 2x2 window; the data flow, op counts and
fan-in/fan-out of the pyramid are kept, the exact coordinate mapping is
approximated (documented in DESIGN.md).

    python paper_2012_07145_b200/pipelines/make_pipelines.py
"""

from __future__ import annotations

import os

HERE = os.path.dirname(os.path.abspath(__file__))


class P:
    def __init__(self, title):
        self.lines = [f"# {title}"]

    def func(self, name, dims, nbytes=4, external=False):
        d = ", ".join(f"{k}={v}" for k, v in dims)
        self.lines.append("")
        self.lines.append(f"func {name} dims ({d}) bytes {nbytes}" + (" external" if external else ""))

    def stage(self, name, **ops):
        o = " ".join(f"{k}={v}" for k, v in ops.items() if v)
        self.lines.append(f"stage {name}" + (f" ops {o}" if o else ""))

    def read(self, name, producer, *dims):
        """dims: (stride, lo, hi) per dim"""
        w = " ".join(f"dim {n} stride {s} lo {lo} hi {hi}" for n, (s, lo, hi) in zip("xyczw", dims))
        self.lines.append(f"read {name} from {producer} {w}")

    def output(self, name):
        self.lines.append("")
        self.lines.append(f"output {name}")

    def text(self):
        return "\n".join(self.lines) + "\n"


PT = (1, 0, 0)


def unsharp(W=1536, H=2560):
    p = P("Unsharp mask, 3 channels: gray -> separable 5-tap Gaussian -> sharpen ratio -> apply")
    rgb = (("x", W), ("y", H), ("c", 3))
    one = (("x", W), ("y", H), ("c", 1))
    p.func("input", rgb, external=True)
    p.func("gray", one)
    p.stage("gray", add=2, mul=3)
    p.read("gray", "input", PT, PT, (0, 0, 2))
    p.func("blur_y", one)
    p.stage("blur_y", add=4, mul=5)
    p.read("blur_y", "gray", PT, (1, -2, 2), PT)
    p.func("blur_x", one)
    p.stage("blur_x", add=4, mul=5)
    p.read("blur_x", "blur_y", (1, -2, 2), PT, PT)
    p.func("sharpen", one)
    p.stage("sharpen", add=1, mul=2)
    p.read("sharpen", "gray", PT, PT, PT)
    p.read("sharpen", "blur_x", PT, PT, PT)
    p.func("ratio", one)
    p.stage("ratio", div=1, minmax=1)
    p.read("ratio", "sharpen", PT, PT, PT)
    p.read("ratio", "gray", PT, PT, PT)
    p.func("scaled", rgb)
    p.stage("scaled", mul=1)
    p.read("scaled", "ratio", PT, PT, (0, 0, 0))
    p.read("scaled", "input", PT, PT, PT)
    p.func("output", rgb, nbytes=1)
    p.stage("output", minmax=2, cast=1)
    p.read("output", "scaled", PT, PT, PT)
    p.output("output")
    return p.text()


def harris(W=1536, H=2560):
    p = P("Harris corner detector: gray -> Sobel gradients -> structure tensor -> 3x3 box -> response")
    rgb = (("x", W), ("y", H), ("c", 3))
    one = (("x", W), ("y", H), ("c", 1))
    p.func("input", rgb, external=True)
    p.func("gray", one)
    p.stage("gray", add=2, mul=3)
    p.read("gray", "input", PT, PT, (0, 0, 2))
    for g, wx, wy in (("Iy", (1, -1, 1), (1, -1, 1)), ("Ix", (1, -1, 1), (1, -1, 1))):
        p.func(g, one)
        p.stage(g, add=5, mul=6)
        p.read(g, "gray", wx, wy, PT)
    for name, a, b in (("Ixx", "Ix", "Ix"), ("Iyy", "Iy", "Iy"), ("Ixy", "Ix", "Iy")):
        p.func(name, one)
        p.stage(name, mul=1)
        p.read(name, a, PT, PT, PT)
        if b != a:
            p.read(name, b, PT, PT, PT)
    for name, src in (("Sxx", "Ixx"), ("Syy", "Iyy"), ("Sxy", "Ixy")):
        p.func(name, one)
        p.stage(name, add=8)
        p.read(name, src, (1, -1, 1), (1, -1, 1), PT)
    p.func("det", one)
    p.stage("det", add=1, mul=2)
    for s in ("Sxx", "Syy", "Sxy"):
        p.read("det", s, PT, PT, PT)
    p.func("trace", one)
    p.stage("trace", add=1)
    p.read("trace", "Sxx", PT, PT, PT)
    p.read("trace", "Syy", PT, PT, PT)
    p.func("output", one)
    p.stage("output", add=1, mul=2)
    p.read("output", "det", PT, PT, PT)
    p.read("output", "trace", PT, PT, PT)
    p.output("output")
    return p.text()


def resnet_block(S=56, C=256, M=64):
    p = P("ResNet-50 bottleneck block (conv2_x): 1x1 256->64, 3x3 64->64, 1x1 64->256, + identity, ReLU; "
          "channel reductions are stride-0 windows (as pipelines/conv.txt)")
    p.func("input", (("x", S), ("y", S), ("c", C)), external=True)
    p.func("conv1", (("x", S), ("y", S), ("c", M)))
    p.stage("conv1", add=C, mul=C)
    p.read("conv1", "input", PT, PT, (0, 0, C - 1))
    p.func("bn1", (("x", S), ("y", S), ("c", M)))
    p.stage("bn1", add=1, mul=1, minmax=1)
    p.read("bn1", "conv1", PT, PT, PT)
    p.func("conv2", (("x", S), ("y", S), ("c", M)))
    p.stage("conv2", add=9 * M, mul=9 * M)
    p.read("conv2", "bn1", (1, -1, 1), (1, -1, 1), (0, 0, M - 1))
    p.func("bn2", (("x", S), ("y", S), ("c", M)))
    p.stage("bn2", add=1, mul=1, minmax=1)
    p.read("bn2", "conv2", PT, PT, PT)
    p.func("conv3", (("x", S), ("y", S), ("c", C)))
    p.stage("conv3", add=M, mul=M)
    p.read("conv3", "bn2", PT, PT, (0, 0, M - 1))
    p.func("bn3", (("x", S), ("y", S), ("c", C)))
    p.stage("bn3", add=1, mul=1)
    p.read("bn3", "conv3", PT, PT, PT)
    p.func("output", (("x", S), ("y", S), ("c", C)))
    p.stage("output", add=1, minmax=1)
    p.read("output", "bn3", PT, PT, PT)
    p.read("output", "input", PT, PT, PT)
    p.output("output")
    return p.text()


def camera_pipe(W=2560, H=1920):
    """~100 funcs: the Halide camera pipe's stages, with the demosaic's
    per-phase interpolations spelled out per colour plane and a multi-pass
    denoise / sharpen to reach the ~100-stage scale of SURVEY C3.  The
    demosaic funcs carry their full op counts (> CHEAP_INLINE_OPS, as the
    gradient-corrected interpolations of the Halide pipe do), so the
    strided plane reads are not inlined through three levels of fan-in."""
    p = P("Camera pipe: hot-pixel suppression, Bayer deinterleave (stride-2 reads), demosaic, "
          "colour correction, tone curve, multi-pass denoise and sharpening")
    raw = (("x", W), ("y", H))
    half = (("x", W // 2), ("y", H // 2))
    p.func("raw", raw, nbytes=2, external=True)
    p.func("denoised", raw, nbytes=2)
    p.stage("denoised", minmax=8)
    p.read("denoised", "raw", (1, -2, 2), (1, -2, 2))
    planes = []
    for name, ox, oy in (("g_gr", 0, 0), ("r_r", 1, 0), ("b_b", 0, 1), ("g_gb", 1, 1)):
        p.func(name, half, nbytes=2)
        p.stage(name, cast=1, minmax=4, compare=4)   # per-plane clamp / hot-pixel test
        p.read(name, "denoised", (2, ox, ox), (2, oy, oy))
        planes.append(name)
    # demosaic: per-phase interpolations (Halide's demosaic has ~20 funcs)
    interp = []
    for tgt in ("g_r", "g_b", "r_gr", "b_gr", "r_gb", "b_gb", "r_b", "b_r"):
        for pas in ("h", "v"):
            n = f"{tgt}_{pas}"
            p.func(n, half, nbytes=2)
            p.stage(n, add=4, mul=2, div=1, minmax=2)   # gradient-corrected interpolation
            src = planes[(len(interp) + (pas == "v")) % 4]
            win = ((1, -1, 1), (1, 0, 0)) if pas == "h" else ((1, 0, 0), (1, -1, 1))
            p.read(n, src, *win)
            interp.append(n)
        n = f"{tgt}_sel"
        p.func(n, half, nbytes=2)
        p.stage(n, add=3, compare=3, minmax=3)   # pick the direction of least gradient
        p.read(n, f"{tgt}_h", PT, PT)
        p.read(n, f"{tgt}_v", PT, PT)
        interp.append(n)
    chans = []
    for c in ("r", "g", "b"):
        n = f"{c}_full"
        p.func(n, raw, nbytes=2)
        p.stage(n, add=3, compare=2)
        for src in (f"r_gr_sel" if c == "r" else f"b_gr_sel" if c == "b" else "g_r_sel",
                    f"r_b_sel" if c == "r" else f"b_r_sel" if c == "b" else "g_b_sel"):
            p.read(n, src, (1, 0, 1), (1, 0, 1))   # upsample approximated (docstring)
        p.read(n, "denoised", PT, PT)
        chans.append(n)
    # colour correction matrix (3x3) and tone curve per channel
    cc = []
    for c in ("r", "g", "b"):
        n = f"{c}_cc"
        p.func(n, raw, nbytes=4)
        p.stage(n, add=3, mul=3, cast=1)
        for src in chans:
            p.read(n, src, PT, PT)
        cc.append(n)
    prev = cc
    # multi-pass edge-aware denoise (bilateral-ish), per channel
    for it in range(8):
        nxt = []
        for ci, c in enumerate(("r", "g", "b")):
            bx = f"{c}_dn{it}_x"
            p.func(bx, raw, nbytes=4)
            p.stage(bx, add=4, mul=5, transcendental=1)
            p.read(bx, prev[ci], (1, -2, 2), PT)
            by = f"{c}_dn{it}_y"
            p.func(by, raw, nbytes=4)
            p.stage(by, add=4, mul=5, transcendental=1)
            p.read(by, bx, PT, (1, -2, 2))
            p.read(by, prev[ci], PT, PT)
            nxt.append(by)
        prev = nxt
    # luma-based sharpening and tone curve
    p.func("luma", raw, nbytes=4)
    p.stage("luma", add=2, mul=3)
    for src in prev:
        p.read("luma", src, PT, PT)
    p.func("luma_blur_x", raw, nbytes=4)
    p.stage("luma_blur_x", add=2, mul=1)
    p.read("luma_blur_x", "luma", (1, -1, 1), PT)
    p.func("luma_blur", raw, nbytes=4)
    p.stage("luma_blur", add=2, mul=1)
    p.read("luma_blur", "luma_blur_x", PT, (1, -1, 1))
    outs = []
    for ci, c in enumerate(("r", "g", "b")):
        n = f"{c}_sharp"
        p.func(n, raw, nbytes=4)
        p.stage(n, add=2, mul=2)
        p.read(n, prev[ci], PT, PT)
        p.read(n, "luma", PT, PT)
        p.read(n, "luma_blur", PT, PT)
        t = f"{c}_curve"
        p.func(t, raw, nbytes=1)
        p.stage(t, transcendental=1, minmax=2, cast=1)
        p.read(t, n, PT, PT)
        outs.append(t)
    p.func("output", raw, nbytes=1)
    p.stage("output", cast=1)
    for o in outs:
        p.read("output", o, PT, PT)
    p.output("output")
    return p.text()


def local_laplacian(W=1536, H=2560, levels=8, k=4):
    """Gaussian pyramid of the input, k intensity levels processed per
    pyramid level (the remapping LUT), Laplacian pyramid, collapse."""
    p = P(f"Local Laplacian filter: {levels}-level pyramids, {k} intensity levels "
          "(upsampling approximated by same-size expanded funcs, see module docstring)")
    dims = [(("x", max(1, W >> l)), ("y", max(1, H >> l))) for l in range(levels)]
    p.func("input", dims[0], nbytes=2, external=True)
    p.func("gray", dims[0])
    p.stage("gray", cast=1, mul=1)
    p.read("gray", "input", PT, PT)
    # remapped images per intensity level, then their Gaussian pyramids
    gpyr = {}
    for j in range(k):
        n = f"remap{j}"
        p.func(n, dims[0])
        p.stage(n, add=2, mul=3, transcendental=1)
        p.read(n, "gray", PT, PT)
        gpyr[(j, 0)] = n
    p.func("g0", dims[0])
    p.stage("g0", mul=1)
    p.read("g0", "gray", PT, PT)
    ipyr = {0: "g0"}
    for l in range(1, levels):
        for j in list(range(k)) + [None]:
            src = ipyr[l - 1] if j is None else gpyr[(j, l - 1)]
            dx = f"{'g' if j is None else f'r{j}_'}dx{l}"
            p.func(dx, (dims[l][0], dims[l - 1][1]))
            p.stage(dx, add=4, mul=2)
            p.read(dx, src, (2, -1, 2), PT)
            dn = f"{'g' if j is None else f'r{j}_'}d{l}"
            p.func(dn, dims[l])
            p.stage(dn, add=4, mul=2)
            p.read(dn, dx, PT, (2, -1, 2))
            if j is None:
                ipyr[l] = dn
            else:
                gpyr[(j, l)] = dn
    # Laplacian of the selected intensity level at each pyramid level
    lap = {}
    for l in range(levels - 1):
        n = f"lap{l}"
        p.func(n, dims[l])
        p.stage(n, add=k + 1, mul=k, compare=k)
        p.read(n, ipyr[l], PT, PT)
        for j in range(k):
            p.read(n, gpyr[(j, l)], PT, PT)
        lap[l] = n
    # collapse: the coarsest output level blends the intensity levels'
    # tops, then coarse-to-fine: expanded coarse level + Laplacian
    top = f"base{levels - 1}"
    p.func(top, dims[levels - 1])
    p.stage(top, add=k, mul=k)
    for j in range(k):
        p.read(top, gpyr[(j, levels - 1)], PT, PT)
    cur = top
    for l in range(levels - 2, -1, -1):
        e = f"expand{l}"
        p.func(e, dims[l])
        p.stage(e, add=3, mul=4)
        p.read(e, cur, (1, 0, 1), (1, 0, 1))   # upsample approximated, see docstring
        c = f"col{l}"
        p.func(c, dims[l])
        p.stage(c, add=1)
        p.read(c, e, PT, PT)
        p.read(c, lap[l], PT, PT)
        cur = c
    p.func("output", dims[0], nbytes=2)
    p.stage("output", cast=1, minmax=2)
    p.read("output", cur, PT, PT)
    p.read("output", "input", PT, PT)
    p.output("output")
    return p.text()


BUILDERS = {"unsharp": unsharp, "harris": harris, "resnet_block": resnet_block,
            # the reference's brute-force lane-address emulation runs out of
            # memory on 256-channel windows; this scaled block is the one
            # golden fixtures are recorded on (same structure, 32/8 channels)
            "resnet_small": lambda: resnet_block(S=28, C=32, M=8),
            "camera_pipe": camera_pipe, "local_laplacian": local_laplacian}


def main():
    for name, fn in BUILDERS.items():
        with open(os.path.join(HERE, f"{name}.txt"), "w") as fh:
            fh.write(fn())


if __name__ == "__main__":
    main()
