"""SparkNet's data-parallel hot path (arXiv:1511.06051), B200-native.

Each of K workers (one per GPU) runs tau local minibatch SGD steps of a Caffe-style CNN
on its own HBM-resident shard; the driver then averages the K workers' weights with one
collective over NVLink.  The compute path is libpsg.so (hand-written sm_100a CUDA behind
the C ABI in include/psg.h); this package is the host mirror of the reference's C++ API
(/root/reference/proj/include/parasgd: net_spec.hpp, model.hpp, weights.hpp, data.hpp,
schemes.hpp).  Importing the package does not load the native library; the first device
call does, and fails loudly if it is missing (there is no CPU fallback).
"""
from . import netspec
from .netspec import (LayerSpec, NetSpec, conv_layer, data_layer, dropout_layer, label_layer,
                      linear_layer, lrn_layer, make_alexnet, make_cifar10_quick, make_cq_valid,
                      make_lenet_small, make_mlp, pool_layer, relu_layer, softmax_loss_layer)
from .weights import WeightCollection, weights_mean

__all__ = [
    "netspec", "LayerSpec", "NetSpec", "conv_layer", "data_layer", "dropout_layer",
    "label_layer", "linear_layer", "lrn_layer", "make_alexnet", "make_cifar10_quick",
    "make_cq_valid", "make_lenet_small", "make_mlp", "pool_layer", "relu_layer",
    "softmax_loss_layer", "WeightCollection", "weights_mean",
]
