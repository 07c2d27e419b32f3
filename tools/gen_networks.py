"""Generate the benchmark networks as pipeline-spec (.pl) files.

The reference ships only toy/train/deep assets (pkg/assets/pipelines); the
BASELINE configs name VGG-16, ResNet-18, ResNet-50 and MobileNet-v2 plus a
2-D conv3x3+ReLU+maxpool chain.  These are written in the reference's text
format (pipeline_ir.py:347-352) with the conventions of SURVEY.md Appendix A:

* valid (unpadded) convolutions: `reduce ci:Cin`, flops 2*k*k,
  `in src map ci*1+1, y*s+k, x*s+k` and a weight buffer
  `in W map co*1+1, ci*1+1, _*0+k, _*0+k`;
* pointwise stages use identity maps, max-pool `y*s+k`;
* residual adds read both inputs with identity maps (skip corner-cropped);
* depthwise convs have no reduction dim;
* head: global average pool `reduce y,x`, then FC `reduce i`.

Run: python tools/gen_networks.py  (writes assets/pipelines/nets/*.pl)
"""

from __future__ import annotations

import pathlib


class Net:
    def __init__(self, name, c, h, w):
        self.name = name
        self.buffers = []
        self.stages = []
        self.buffers.append(f"buffer input dims {c}x{h}x{w} elem 4")
        self.shape = {"input": (c, h, w)}
        self.n = 0

    def _uid(self, base):
        self.n += 1
        return f"{base}{self.n}"

    def conv(self, src, cout, k, s=1, base="conv"):
        cin, h, w = self.shape[src]
        ho, wo = (h - k) // s + 1, (w - k) // s + 1
        name = self._uid(base)
        wname = name + "_w"
        self.buffers.append(f"buffer {wname} dims {cout}x{cin}x{k}x{k} elem 4")
        self.stages.append(
            f"stage {name} dims co:{cout},y:{ho},x:{wo} reduce ci:{cin} flops {2 * k * k}\n"
            f"  in {src} map ci*1+1, y*{s}+{k}, x*{s}+{k}\n"
            f"  in {wname} map co*1+1, ci*1+1, _*0+{k}, _*0+{k}"
        )
        self.shape[name] = (cout, ho, wo)
        return name

    def dwconv(self, src, k, s=1):
        c, h, w = self.shape[src]
        ho, wo = (h - k) // s + 1, (w - k) // s + 1
        name = self._uid("dw")
        wname = name + "_w"
        self.buffers.append(f"buffer {wname} dims {c}x{k}x{k} elem 4")
        self.stages.append(
            f"stage {name} dims c:{c},y:{ho},x:{wo} flops {2 * k * k}\n"
            f"  in {src} map c*1+1, y*{s}+{k}, x*{s}+{k}\n"
            f"  in {wname} map c*1+1, _*0+{k}, _*0+{k}"
        )
        self.shape[name] = (c, ho, wo)
        return name

    def relu(self, src):
        c, h, w = self.shape[src]
        name = self._uid("relu")
        self.stages.append(
            f"stage {name} dims c:{c},y:{h},x:{w} flops 1\n"
            f"  in {src} map c*1+1, y*1+1, x*1+1"
        )
        self.shape[name] = (c, h, w)
        return name

    def pool(self, src, k=2, s=2):
        c, h, w = self.shape[src]
        ho, wo = (h - k) // s + 1, (w - k) // s + 1
        name = self._uid("pool")
        self.stages.append(
            f"stage {name} dims c:{c},y:{ho},x:{wo} flops {k * k}\n"
            f"  in {src} map c*1+1, y*{s}+{k}, x*{s}+{k}"
        )
        self.shape[name] = (c, ho, wo)
        return name

    def add(self, a, b):
        c, h, w = self.shape[a]
        name = self._uid("add")
        self.stages.append(
            f"stage {name} dims c:{c},y:{h},x:{w} flops 1\n"
            f"  in {a} map c*1+1, y*1+1, x*1+1\n"
            f"  in {b} map c*1+1, y*1+1, x*1+1"
        )
        self.shape[name] = (c, h, w)
        return name

    def head(self, src, classes, hidden=None):
        c, h, w = self.shape[src]
        gap = self._uid("gap")
        self.stages.append(
            f"stage {gap} dims c:{c} reduce y:{h},x:{w} flops 1\n"
            f"  in {src} map c*1+1, y*1+1, x*1+1"
        )
        self.shape[gap] = (c,)
        cur, width = gap, c
        dims = ([hidden] if hidden else []) + [classes]
        for i, o in enumerate(dims):
            name = self._uid("fc")
            wname = name + "_w"
            self.buffers.append(f"buffer {wname} dims {o}x{width} elem 4")
            out = " output" if i == len(dims) - 1 else ""
            self.stages.append(
                f"stage {name} dims o:{o} reduce i:{width} flops 2{out}\n"
                f"  in {cur} map i*1+1\n"
                f"  in {wname} map o*1+1, i*1+1"
            )
            self.shape[name] = (o,)
            cur, width = name, o
        return cur

    def text(self, comment):
        if not any(" output\n" in st or st.endswith(" output") for st in self.stages):
            head, _, rest = self.stages[-1].partition("\n")
            self.stages[-1] = head + " output" + ("\n" + rest if rest else "")
        lines = [f"# {comment}", f"pipeline {self.name}"]
        lines += self.buffers
        lines += self.stages
        return "\n".join(lines) + "\n"


def vgg16():
    n = Net("vgg16", 3, 252, 252)
    x = "input"
    for i, (reps, ch) in enumerate([(2, 64), (2, 128), (3, 256), (3, 512), (3, 512)]):
        for _ in range(reps):
            x = n.relu(n.conv(x, ch, 3))
        x = n.pool(x)
    x = n.head(x, 1000, hidden=4096)
    return n.text("VGG-16 probe: 13 valid 3x3 convs + ReLU, 5 max-pools, GAP, 2 FC (T=34)")


def resnet18():
    n = Net("resnet18", 3, 544, 544)
    x = n.pool(n.relu(n.conv("input", 64, 7, 2)), 3, 2)
    cin = 64
    for stage, ch in enumerate([64, 128, 256, 512]):
        for blk in range(2):
            s = 2 if (stage > 0 and blk == 0) else 1
            y = n.relu(n.conv(x, ch, 3, s))
            y = n.conv(y, ch, 3, 1)
            skip = x
            if s != 1 or cin != ch:
                skip = n.conv(x, ch, 1, s, base="proj")
            x = n.relu(n.add(y, skip))
            cin = ch
    n.head(x, 1000)
    return n.text("ResNet-18 probe: valid convs, corner-cropped skips, GAP+FC (T=48)")


def resnet50():
    n = Net("resnet50", 3, 544, 544)
    x = n.pool(n.relu(n.conv("input", 64, 7, 2)), 3, 2)
    cin = 64
    for stage, (reps, mid) in enumerate([(3, 64), (4, 128), (6, 256), (3, 512)]):
        out = mid * 4
        for blk in range(reps):
            s = 2 if (stage > 0 and blk == 0) else 1
            y = n.relu(n.conv(x, mid, 1, 1))
            y = n.relu(n.conv(y, mid, 3, s))
            y = n.conv(y, out, 1, 1)
            skip = x
            if s != 1 or cin != out:
                skip = n.conv(x, out, 1, s, base="proj")
            x = n.relu(n.add(y, skip))
            cin = out
    n.head(x, 1000)
    return n.text("ResNet-50 probe: bottleneck blocks, valid convs, GAP+FC (T=121)")


def mobilenet_v2():
    n = Net("mobilenet_v2", 3, 672, 672)
    x = n.relu(n.conv("input", 32, 3, 2))
    cin = 32
    cfg = [(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2),
           (6, 96, 3, 1), (6, 160, 3, 2), (6, 320, 1, 1)]
    for t, c, reps, s0 in cfg:
        for r in range(reps):
            s = s0 if r == 0 else 1
            y = x
            if t != 1:
                y = n.relu(n.conv(y, cin * t, 1, 1, base="expand"))
            y = n.relu(n.dwconv(y, 3, s))
            y = n.conv(y, c, 1, 1, base="project")
            if s == 1 and cin == c:
                y = n.add(y, x)
            x = y
            cin = c
    x = n.relu(n.conv(x, 1280, 1, 1))
    n.head(x, 1000)
    return n.text("MobileNet-v2 probe: inverted residuals, valid depthwise convs (T=99)")


def conv_relu_pool_2d():
    n = Net("crp2d", 3, 66, 66)
    x = n.pool(n.relu(n.conv("input", 16, 3)))
    lines = n.text("3-layer conv3x3 + ReLU + 2x2 maxpool, 2-D (configs[0] 2-D variant)")
    return lines


NETS = {
    "vgg16": vgg16,
    "resnet18": resnet18,
    "resnet50": resnet50,
    "mobilenet_v2": mobilenet_v2,
    "crp2d": conv_relu_pool_2d,
}


def main():
    out = pathlib.Path(__file__).resolve().parent.parent / "assets" / "pipelines" / "nets"
    out.mkdir(parents=True, exist_ok=True)
    for name, fn in NETS.items():
        (out / f"{name}.pl").write_text(fn())
        print("wrote", out / f"{name}.pl")


if __name__ == "__main__":
    main()
