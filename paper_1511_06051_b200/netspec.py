"""Declarative layer graphs: the host-side mirror of ``net_spec.hpp``.

``LayerSpec`` / ``NetSpec`` and the factory helpers follow
/root/reference/proj/include/parasgd/net_spec.hpp:28-177 (same names, same
argument meaning, same validation errors as ``ValueError`` <-> std::invalid_argument).
The Caffe geometry fields (pad, stride, group, AVE/ceil pooling, LRN, dropout,
multipliers) are additive extensions whose defaults reproduce the reference.

``NetSpec.to_c()`` packs the graph into the ``psg_layer_desc`` array that the
C ABI (include/psg.h) consumes.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Sequence

# psg_layer_kind (include/psg.h) <-> LayerKind (net_spec.hpp:11)
DATA, LABEL, CONV, POOL, LINEAR, RELU, SOFTMAX_LOSS, LRN, DROPOUT, CONCAT = range(10)
POOL_MAX, POOL_AVE = 0, 1
KIND_NAMES = {DATA: "data", LABEL: "label", CONV: "conv", POOL: "pool", LINEAR: "linear",
              RELU: "relu", SOFTMAX_LOSS: "softmax", LRN: "lrn", DROPOUT: "dropout",
              CONCAT: "concat"}


class CLayerDesc(ctypes.Structure):
    """ctypes mirror of ``psg_layer_desc`` (include/psg.h)."""
    _fields_ = [
        ("kind", ctypes.c_int),
        ("name", ctypes.c_char * 48),
        ("n_inputs", ctypes.c_int),
        ("inputs", ctypes.c_int * 8),
        ("batch", ctypes.c_int), ("channels", ctypes.c_int),
        ("height", ctypes.c_int), ("width", ctypes.c_int),
        ("num_output", ctypes.c_int),
        ("kernel_h", ctypes.c_int), ("kernel_w", ctypes.c_int),
        ("stride_h", ctypes.c_int), ("stride_w", ctypes.c_int),
        ("pad_h", ctypes.c_int), ("pad_w", ctypes.c_int),
        ("group", ctypes.c_int),
        ("pool", ctypes.c_int),
        ("ceil_mode", ctypes.c_int),
        ("local_size", ctypes.c_int),
        ("alpha", ctypes.c_double), ("beta", ctypes.c_double), ("k", ctypes.c_double),
        ("dropout_ratio", ctypes.c_double),
        ("loss_weight", ctypes.c_double),
        ("lr_mult_w", ctypes.c_double), ("lr_mult_b", ctypes.c_double),
        ("decay_mult_w", ctypes.c_double), ("decay_mult_b", ctypes.c_double),
    ]


@dataclass
class LayerSpec:
    """net_spec.hpp:28-38 plus Caffe geometry."""
    kind: int = DATA
    name: str = ""
    inputs: List[str] = field(default_factory=list)
    shape: List[int] = field(default_factory=list)   # data: [b,c,h,w]; label: [b,1]
    kernel_h: int = 0
    kernel_w: int = 0
    num_filters: int = 0                              # conv
    stride_h: int = 1
    stride_w: int = 1
    num_outputs: int = 0                              # linear
    pad_h: int = 0
    pad_w: int = 0
    group: int = 1
    pool: int = POOL_MAX
    ceil_mode: bool = False
    local_size: int = 5
    alpha: float = 1e-4
    beta: float = 0.75
    k: float = 1.0
    dropout_ratio: float = 0.5
    loss_weight: float = 1.0
    lr_mult_w: float = 1.0
    lr_mult_b: float = 1.0
    decay_mult_w: float = 1.0
    decay_mult_b: float = 1.0


def data_layer(name: str, batch: int, c: int, h: int, w: int) -> LayerSpec:
    return LayerSpec(kind=DATA, name=name, shape=[batch, c, h, w])


def label_layer(name: str, batch: int) -> LayerSpec:
    return LayerSpec(kind=LABEL, name=name, shape=[batch, 1])


def conv_layer(name: str, input: str, kh: int, kw: int, num_filters: int, *, stride: int = 1,
               pad: int = 0, group: int = 1, lr_mult=(1.0, 1.0), decay_mult=(1.0, 1.0)) -> LayerSpec:
    return LayerSpec(kind=CONV, name=name, inputs=[input], kernel_h=kh, kernel_w=kw,
                     num_filters=num_filters, stride_h=stride, stride_w=stride, pad_h=pad,
                     pad_w=pad, group=group, lr_mult_w=lr_mult[0], lr_mult_b=lr_mult[1],
                     decay_mult_w=decay_mult[0], decay_mult_b=decay_mult[1])


def pool_layer(name: str, input: str, kh: int, kw: int, sh: int, sw: int, *,
               method: int = POOL_MAX, pad: int = 0, ceil_mode: bool = False) -> LayerSpec:
    return LayerSpec(kind=POOL, name=name, inputs=[input], kernel_h=kh, kernel_w=kw,
                     stride_h=sh, stride_w=sw, pool=method, pad_h=pad, pad_w=pad,
                     ceil_mode=ceil_mode)


def linear_layer(name: str, input: str, num_outputs: int, *, lr_mult=(1.0, 1.0),
                 decay_mult=(1.0, 1.0)) -> LayerSpec:
    return LayerSpec(kind=LINEAR, name=name, inputs=[input], num_outputs=num_outputs,
                     lr_mult_w=lr_mult[0], lr_mult_b=lr_mult[1], decay_mult_w=decay_mult[0],
                     decay_mult_b=decay_mult[1])


def relu_layer(name: str, input: str) -> LayerSpec:
    return LayerSpec(kind=RELU, name=name, inputs=[input])


def lrn_layer(name: str, input: str, local_size: int = 5, alpha: float = 1e-4,
              beta: float = 0.75, k: float = 1.0) -> LayerSpec:
    return LayerSpec(kind=LRN, name=name, inputs=[input], local_size=local_size, alpha=alpha,
                     beta=beta, k=k)


def dropout_layer(name: str, input: str, ratio: float = 0.5) -> LayerSpec:
    return LayerSpec(kind=DROPOUT, name=name, inputs=[input], dropout_ratio=ratio)


def concat_layer(name: str, inputs: Sequence[str]) -> LayerSpec:
    """Caffe Concat along channels (extension; GoogLeNet inception outputs)."""
    return LayerSpec(kind=CONCAT, name=name, inputs=list(inputs))


def softmax_loss_layer(name: str, logits: str, label: str, loss_weight: float = 1.0) -> LayerSpec:
    return LayerSpec(kind=SOFTMAX_LOSS, name=name, inputs=[logits, label], loss_weight=loss_weight)


@dataclass
class NetSpec:
    """net_spec.hpp:107-177."""
    layers: List[LayerSpec] = field(default_factory=list)

    def validate(self) -> None:
        seen = set()
        n_data = n_label = n_loss = 0
        for l in self.layers:
            if not l.name:
                raise ValueError("net: layer with empty name")
            if l.name in seen:
                raise ValueError(f"net: duplicate layer name '{l.name}'")
            for i in l.inputs:
                if i not in seen:
                    raise ValueError(f"net: layer '{l.name}' references '{i}' which is not "
                                     "declared earlier")
            seen.add(l.name)
            if l.kind == DATA:
                n_data += 1
                if len(l.shape) != 4:
                    raise ValueError("net: data layer needs [b,c,h,w]")
            elif l.kind == LABEL:
                n_label += 1
                if len(l.shape) != 2 or l.shape[1] != 1:
                    raise ValueError("net: label layer needs [b,1]")
            elif l.kind == CONV:
                if len(l.inputs) != 1:
                    raise ValueError("net: conv takes one input")
                if l.kernel_h < 1 or l.kernel_w < 1 or l.num_filters < 1:
                    raise ValueError(f"net: conv '{l.name}' has non-positive geometry")
                if l.stride_h < 1 or l.stride_w < 1 or l.pad_h < 0 or l.pad_w < 0 or l.group < 1:
                    raise ValueError(f"net: conv '{l.name}' has non-positive geometry")
            elif l.kind == POOL:
                if len(l.inputs) != 1:
                    raise ValueError("net: pool takes one input")
                if l.kernel_h < 1 or l.kernel_w < 1 or l.stride_h < 1 or l.stride_w < 1:
                    raise ValueError(f"net: pool '{l.name}' has non-positive geometry")
            elif l.kind == LINEAR:
                if len(l.inputs) != 1:
                    raise ValueError("net: linear takes one input")
                if l.num_outputs < 1:
                    raise ValueError(f"net: linear '{l.name}' needs positive outputs")
            elif l.kind in (RELU, LRN, DROPOUT):
                if len(l.inputs) != 1:
                    raise ValueError(f"net: {KIND_NAMES[l.kind]} takes one input")
                if l.kind == LRN and (l.local_size < 1 or l.local_size % 2 == 0):
                    raise ValueError("net: lrn local_size must be odd")
                if l.kind == DROPOUT and not (0.0 <= l.dropout_ratio < 1.0):
                    raise ValueError("net: dropout ratio must be in [0,1)")
            elif l.kind == SOFTMAX_LOSS:
                n_loss += 1
                if len(l.inputs) != 2:
                    raise ValueError("net: softmax loss takes [logits, label]")
            elif l.kind == CONCAT:
                if not 1 <= len(l.inputs) <= 8:
                    raise ValueError("net: concat takes 1..8 inputs")
            else:
                raise ValueError(f"net: unknown layer kind {l.kind}")
        if n_data != 1:
            raise ValueError("net: exactly one data layer required")
        if n_label != 1:
            raise ValueError("net: exactly one label layer required")
        if n_loss < 1:  # several weighted losses: auxiliary heads (extension)
            raise ValueError("net: at least one softmax loss layer required")

    def data_spec(self) -> LayerSpec:
        for l in self.layers:
            if l.kind == DATA:
                return l
        raise RuntimeError("net: no data layer")

    def index_of(self, name: str) -> int:
        for i, l in enumerate(self.layers):
            if l.name == name:
                return i
        raise ValueError(f"net: unknown layer '{name}'")

    def to_c(self):
        """Pack into a ``psg_layer_desc[n]`` ctypes array."""
        self.validate()
        arr = (CLayerDesc * len(self.layers))()
        for i, l in enumerate(self.layers):
            d = arr[i]
            d.kind = l.kind
            d.name = l.name.encode()[:47]
            d.n_inputs = len(l.inputs)
            for j, name in enumerate(l.inputs):
                d.inputs[j] = self.index_of(name)
            if l.kind == DATA:
                d.batch, d.channels, d.height, d.width = l.shape
            elif l.kind == LABEL:
                d.batch = l.shape[0]
            d.num_output = l.num_filters if l.kind == CONV else l.num_outputs
            d.kernel_h, d.kernel_w = l.kernel_h, l.kernel_w
            d.stride_h, d.stride_w = l.stride_h, l.stride_w
            d.pad_h, d.pad_w = l.pad_h, l.pad_w
            d.group = l.group
            d.pool = l.pool
            d.ceil_mode = int(l.ceil_mode)
            d.local_size = l.local_size
            d.alpha, d.beta, d.k = l.alpha, l.beta, l.k
            d.dropout_ratio = l.dropout_ratio
            d.loss_weight = l.loss_weight
            d.lr_mult_w, d.lr_mult_b = l.lr_mult_w, l.lr_mult_b
            d.decay_mult_w, d.decay_mult_b = l.decay_mult_w, l.decay_mult_b
        return arr

    def is_reference_expressible(self) -> bool:
        """True when the unmodified reference (net_spec.hpp) can build this graph."""
        for l in self.layers:
            if l.kind in (LRN, DROPOUT, CONCAT):
                return False
            if l.kind == CONV and (l.pad_h or l.pad_w or l.stride_h != 1 or l.stride_w != 1
                                   or l.group != 1):
                return False
            if l.kind == POOL and (l.pool != POOL_MAX or l.ceil_mode or l.pad_h or l.pad_w):
                return False
            if l.kind == SOFTMAX_LOSS and l.loss_weight != 1.0:
                return False
        if sum(l.kind == SOFTMAX_LOSS for l in self.layers) != 1:
            return False
        return True


# ---------------------------------------------------------------- presets ----
def make_lenet_small(batch: int, c: int, h: int, w: int, num_classes: int) -> NetSpec:
    """net_spec.hpp:182-199."""
    net = NetSpec([
        data_layer("data", batch, c, h, w),
        label_layer("label", batch),
        conv_layer("conv1", "data", 5, 5, 8),
        pool_layer("pool1", "conv1", 2, 2, 2, 2),
        conv_layer("conv2", "pool1", 5, 5, 16),
        pool_layer("pool2", "conv2", 2, 2, 2, 2),
        linear_layer("ip1", "pool2", 64),
        relu_layer("relu1", "ip1"),
        linear_layer("ip2", "relu1", num_classes),
        softmax_loss_layer("loss", "ip2", "label"),
    ])
    net.validate()
    return net


def make_mlp(batch: int, c: int, h: int, w: int, num_classes: int, hidden: int = 64) -> NetSpec:
    """net_spec.hpp:202-215."""
    net = NetSpec([
        data_layer("data", batch, c, h, w),
        label_layer("label", batch),
        linear_layer("ip1", "data", hidden),
        relu_layer("relu1", "ip1"),
        linear_layer("ip2", "relu1", num_classes),
        softmax_loss_layer("loss", "ip2", "label"),
    ])
    net.validate()
    return net


def make_cq_valid(batch: int, num_classes: int = 10) -> NetSpec:
    """SURVEY §8(d) `cq-valid`: the cifar10_quick analog the unmodified reference can express."""
    net = NetSpec([
        data_layer("data", batch, 3, 32, 32),
        label_layer("label", batch),
        conv_layer("conv1", "data", 5, 5, 32),
        pool_layer("pool1", "conv1", 3, 3, 2, 2),
        relu_layer("relu1", "pool1"),
        conv_layer("conv2", "relu1", 5, 5, 32),
        relu_layer("relu2", "conv2"),
        pool_layer("pool2", "relu2", 3, 3, 2, 2),
        conv_layer("conv3", "pool2", 3, 3, 64),
        relu_layer("relu3", "conv3"),
        linear_layer("ip1", "relu3", 64),
        linear_layer("ip2", "ip1", num_classes),
        softmax_loss_layer("loss", "ip2", "label"),
    ])
    net.validate()
    return net


def make_cifar10_quick(batch: int = 100, num_classes: int = 10) -> NetSpec:
    """Caffe examples/cifar10/cifar10_quick_train_test.prototxt geometry (SURVEY §2.2 "cq"):
    conv 5x5 pad 2 (32, 32, 64), pools 3x3/2 ceil (MAX, AVE, AVE), ip1 64, ip2 10.
    Bias lr_mult 2 as in the prototxt."""
    net = NetSpec([
        data_layer("data", batch, 3, 32, 32),
        label_layer("label", batch),
        conv_layer("conv1", "data", 5, 5, 32, pad=2, lr_mult=(1.0, 2.0)),
        pool_layer("pool1", "conv1", 3, 3, 2, 2, method=POOL_MAX, ceil_mode=True),
        relu_layer("relu1", "pool1"),
        conv_layer("conv2", "relu1", 5, 5, 32, pad=2, lr_mult=(1.0, 2.0)),
        relu_layer("relu2", "conv2"),
        pool_layer("pool2", "relu2", 3, 3, 2, 2, method=POOL_AVE, ceil_mode=True),
        conv_layer("conv3", "pool2", 5, 5, 64, pad=2, lr_mult=(1.0, 2.0)),
        relu_layer("relu3", "conv3"),
        pool_layer("pool3", "relu3", 3, 3, 2, 2, method=POOL_AVE, ceil_mode=True),
        linear_layer("ip1", "pool3", 64, lr_mult=(1.0, 2.0)),
        linear_layer("ip2", "ip1", num_classes, lr_mult=(1.0, 2.0)),
        softmax_loss_layer("loss", "ip2", "label"),
    ])
    net.validate()
    return net


def make_alexnet(batch: int = 256, num_classes: int = 1000) -> NetSpec:
    """BVLC AlexNet (models/bvlc_alexnet/train_val.prototxt): conv1 11x11/4 -> relu -> LRN ->
    max 3/2 -> conv2 5x5 p2 g2 -> relu -> LRN -> max 3/2 -> conv3 3x3 p1 -> conv4 g2 ->
    conv5 g2 -> max 3/2 -> fc6 4096 -> drop -> fc7 4096 -> drop -> fc8.  Bias lr_mult 2,
    decay_mult 0 as in the prototxt."""
    b = dict(lr_mult=(1.0, 2.0), decay_mult=(1.0, 0.0))
    net = NetSpec([
        data_layer("data", batch, 3, 227, 227),
        label_layer("label", batch),
        conv_layer("conv1", "data", 11, 11, 96, stride=4, **b),
        relu_layer("relu1", "conv1"),
        lrn_layer("norm1", "relu1", 5, 1e-4, 0.75),
        pool_layer("pool1", "norm1", 3, 3, 2, 2, ceil_mode=True),
        conv_layer("conv2", "pool1", 5, 5, 256, pad=2, group=2, **b),
        relu_layer("relu2", "conv2"),
        lrn_layer("norm2", "relu2", 5, 1e-4, 0.75),
        pool_layer("pool2", "norm2", 3, 3, 2, 2, ceil_mode=True),
        conv_layer("conv3", "pool2", 3, 3, 384, pad=1, **b),
        relu_layer("relu3", "conv3"),
        conv_layer("conv4", "relu3", 3, 3, 384, pad=1, group=2, **b),
        relu_layer("relu4", "conv4"),
        conv_layer("conv5", "relu4", 3, 3, 256, pad=1, group=2, **b),
        relu_layer("relu5", "conv5"),
        pool_layer("pool5", "relu5", 3, 3, 2, 2, ceil_mode=True),
        linear_layer("fc6", "pool5", 4096, **b),
        relu_layer("relu6", "fc6"),
        dropout_layer("drop6", "relu6", 0.5),
        linear_layer("fc7", "drop6", 4096, **b),
        relu_layer("relu7", "fc7"),
        dropout_layer("drop7", "relu7", 0.5),
        linear_layer("fc8", "drop7", num_classes, **b),
        softmax_loss_layer("loss", "fc8", "label"),
    ])
    net.validate()
    return net


def _inception(layers, name, inp, c1, c3r, c3, c5r, c5, cp, b):
    """One GoogLeNet inception module (bvlc_googlenet): 1x1 | 1x1->3x3 | 1x1->5x5 |
    maxpool 3/1 -> 1x1, each conv followed by ReLU, concatenated along channels."""
    p = name + "/"
    layers += [conv_layer(p + "1x1", inp, 1, 1, c1, **b), relu_layer(p + "relu_1x1", p + "1x1"),
               conv_layer(p + "3x3_reduce", inp, 1, 1, c3r, **b),
               relu_layer(p + "relu_3x3_reduce", p + "3x3_reduce"),
               conv_layer(p + "3x3", p + "relu_3x3_reduce", 3, 3, c3, pad=1, **b),
               relu_layer(p + "relu_3x3", p + "3x3"),
               conv_layer(p + "5x5_reduce", inp, 1, 1, c5r, **b),
               relu_layer(p + "relu_5x5_reduce", p + "5x5_reduce"),
               conv_layer(p + "5x5", p + "relu_5x5_reduce", 5, 5, c5, pad=2, **b),
               relu_layer(p + "relu_5x5", p + "5x5"),
               pool_layer(p + "pool", inp, 3, 3, 1, 1, pad=1, ceil_mode=True),
               conv_layer(p + "pool_proj", p + "pool", 1, 1, cp, **b),
               relu_layer(p + "relu_pool_proj", p + "pool_proj"),
               concat_layer(p + "output", [p + "relu_1x1", p + "relu_3x3", p + "relu_5x5",
                                           p + "relu_pool_proj"])]
    return p + "output"


def _aux_head(layers, name, inp, num_classes, b):
    """GoogLeNet auxiliary classifier (loss weight 0.3)."""
    p = name + "/"
    layers += [pool_layer(p + "ave_pool", inp, 5, 5, 3, 3, method=POOL_AVE, ceil_mode=True),
               conv_layer(p + "conv", p + "ave_pool", 1, 1, 128, **b),
               relu_layer(p + "relu_conv", p + "conv"),
               linear_layer(p + "fc", p + "relu_conv", 1024, **b),
               relu_layer(p + "relu_fc", p + "fc"),
               dropout_layer(p + "drop_fc", p + "relu_fc", 0.7),
               linear_layer(p + "classifier", p + "drop_fc", num_classes, **b),
               softmax_loss_layer(p + "loss", p + "classifier", "label", loss_weight=0.3)]


def make_googlenet(batch: int, num_classes: int = 1000, image: int = 224) -> NetSpec:
    """GoogLeNet (Caffe bvlc_googlenet, with both auxiliary heads at loss weight 0.3):
    conv 7x7/2 -> max 3/2 -> LRN -> 1x1 -> 3x3 -> LRN -> max 3/2 -> inception 3a,3b ->
    max 3/2 -> 4a (aux1) 4b 4c 4d (aux2) 4e -> max 3/2 -> 5a 5b -> ave 7/1 -> drop 0.4 ->
    classifier.  Bias lr_mult 2 / decay_mult 0 as in the prototxt."""
    b = dict(lr_mult=(1.0, 2.0), decay_mult=(1.0, 0.0))
    L = [data_layer("data", batch, 3, image, image), label_layer("label", batch),
         conv_layer("conv1/7x7_s2", "data", 7, 7, 64, stride=2, pad=3, **b),
         relu_layer("conv1/relu_7x7", "conv1/7x7_s2"),
         pool_layer("pool1/3x3_s2", "conv1/relu_7x7", 3, 3, 2, 2, ceil_mode=True),
         lrn_layer("pool1/norm1", "pool1/3x3_s2", 5, 1e-4, 0.75),
         conv_layer("conv2/3x3_reduce", "pool1/norm1", 1, 1, 64, **b),
         relu_layer("conv2/relu_3x3_reduce", "conv2/3x3_reduce"),
         conv_layer("conv2/3x3", "conv2/relu_3x3_reduce", 3, 3, 192, pad=1, **b),
         relu_layer("conv2/relu_3x3", "conv2/3x3"),
         lrn_layer("conv2/norm2", "conv2/relu_3x3", 5, 1e-4, 0.75),
         pool_layer("pool2/3x3_s2", "conv2/norm2", 3, 3, 2, 2, ceil_mode=True)]
    x = _inception(L, "inception_3a", "pool2/3x3_s2", 64, 96, 128, 16, 32, 32, b)
    x = _inception(L, "inception_3b", x, 128, 128, 192, 32, 96, 64, b)
    L.append(pool_layer("pool3/3x3_s2", x, 3, 3, 2, 2, ceil_mode=True))
    x = _inception(L, "inception_4a", "pool3/3x3_s2", 192, 96, 208, 16, 48, 64, b)
    _aux_head(L, "loss1", x, num_classes, b)
    x = _inception(L, "inception_4b", x, 160, 112, 224, 24, 64, 64, b)
    x = _inception(L, "inception_4c", x, 128, 128, 256, 24, 64, 64, b)
    x = _inception(L, "inception_4d", x, 112, 144, 288, 32, 64, 64, b)
    _aux_head(L, "loss2", x, num_classes, b)
    x = _inception(L, "inception_4e", x, 256, 160, 320, 32, 128, 128, b)
    L.append(pool_layer("pool4/3x3_s2", x, 3, 3, 2, 2, ceil_mode=True))
    x = _inception(L, "inception_5a", "pool4/3x3_s2", 256, 160, 320, 32, 128, 128, b)
    x = _inception(L, "inception_5b", x, 384, 192, 384, 48, 128, 128, b)
    L += [pool_layer("pool5/7x7_s1", x, 7, 7, 1, 1, method=POOL_AVE),
          dropout_layer("pool5/drop_7x7_s1", "pool5/7x7_s1", 0.4),
          linear_layer("loss3/classifier", "pool5/drop_7x7_s1", num_classes, **b),
          softmax_loss_layer("loss3/loss3", "loss3/classifier", "label", loss_weight=1.0)]
    net = NetSpec(L)
    net.validate()
    return net


PRESETS = {
    "lenet-small": lambda b, c, h, w, k: make_lenet_small(b, c, h, w, k),
    "mlp": lambda b, c, h, w, k: make_mlp(b, c, h, w, k),
}


def param_count(spec: NetSpec) -> int:
    """P by shape inference (mirrors model.hpp:200-283 plus Caffe geometry)."""
    dims = {}
    total = 0
    for l in spec.layers:
        if l.kind == DATA:
            dims[l.name] = tuple(l.shape[1:])
            continue
        if l.kind == LABEL:
            dims[l.name] = (1, 1, 1)
            continue
        c, h, w = dims[l.inputs[0]]
        if l.kind == CONV:
            oh = (h + 2 * l.pad_h - l.kernel_h) // l.stride_h + 1
            ow = (w + 2 * l.pad_w - l.kernel_w) // l.stride_w + 1
            total += l.num_filters * (c // l.group) * l.kernel_h * l.kernel_w + l.num_filters
            dims[l.name] = (l.num_filters, oh, ow)
        elif l.kind == POOL:
            dims[l.name] = (c, pool_out(h, l.kernel_h, l.stride_h, l.pad_h, l.ceil_mode),
                            pool_out(w, l.kernel_w, l.stride_w, l.pad_w, l.ceil_mode))
        elif l.kind == LINEAR:
            total += l.num_outputs * c * h * w + l.num_outputs
            dims[l.name] = (l.num_outputs, 1, 1)
        elif l.kind == SOFTMAX_LOSS:
            dims[l.name] = (c * h * w, 1, 1)
        elif l.kind == CONCAT:
            dims[l.name] = (sum(dims[i][0] for i in l.inputs), h, w)
        else:
            dims[l.name] = (c, h, w)
    return total


def pool_out(n: int, k: int, s: int, p: int, ceil_mode: bool) -> int:
    if ceil_mode:
        o = -(-(n + 2 * p - k) // s) + 1
        if p > 0 and (o - 1) * s >= n + p:
            o -= 1
        return o
    return (n + 2 * p - k) // s + 1


def forward_macs(spec: NetSpec) -> dict:
    """Per-layer forward multiply-accumulates per image (BASELINE.md §3 work units)."""
    dims = {}
    macs = {}
    for l in spec.layers:
        if l.kind == DATA:
            dims[l.name] = tuple(l.shape[1:])
            continue
        if l.kind == LABEL:
            dims[l.name] = (1, 1, 1)
            continue
        c, h, w = dims[l.inputs[0]]
        if l.kind == CONV:
            oh = (h + 2 * l.pad_h - l.kernel_h) // l.stride_h + 1
            ow = (w + 2 * l.pad_w - l.kernel_w) // l.stride_w + 1
            macs[l.name] = l.num_filters * (c // l.group) * l.kernel_h * l.kernel_w * oh * ow
            dims[l.name] = (l.num_filters, oh, ow)
        elif l.kind == POOL:
            dims[l.name] = (c, pool_out(h, l.kernel_h, l.stride_h, l.pad_h, l.ceil_mode),
                            pool_out(w, l.kernel_w, l.stride_w, l.pad_w, l.ceil_mode))
        elif l.kind == LINEAR:
            macs[l.name] = l.num_outputs * c * h * w
            dims[l.name] = (l.num_outputs, 1, 1)
        elif l.kind == SOFTMAX_LOSS:
            dims[l.name] = (c * h * w, 1, 1)
        elif l.kind == CONCAT:
            dims[l.name] = (sum(dims[i][0] for i in l.inputs), h, w)
        else:
            dims[l.name] = (c, h, w)
    return macs


def train_flops_per_image(spec: NetSpec) -> float:
    """2 * MAC * (fwd + wgrad + dgrad) minus the first layer's dgrad."""
    macs = forward_macs(spec)
    data = spec.data_spec().name
    total = 0.0
    for l in spec.layers:
        if l.name in macs:
            m = macs[l.name]
            first = l.inputs[0] == data
            total += 2.0 * m * (2 if first else 3)
    return total


def layer_names(spec: NetSpec) -> Sequence[str]:
    return [l.name for l in spec.layers]
