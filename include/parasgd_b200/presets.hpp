// parasgd_b200/presets.hpp — the BASELINE.json networks as psg_layer_desc graphs for the C++
// drop-in (extension: the reference's NetSpec, net_spec.hpp:11-38, cannot express padded /
// strided / grouped convolutions, AVE or ceil-mode pooling, LRN, dropout, concat or several
// weighted losses).  Same graphs as paper_1511_06051_b200/netspec.py (make_cifar10_quick,
// make_alexnet, make_googlenet), which the GPU tests check against the oracle.
#pragma once

#include <psg.h>

#include <stdexcept>
#include <string>
#include <vector>

namespace parasgd {
namespace b200 {

/// Appends layers by name; inputs are resolved to indices of earlier layers.
class DescBuilder {
 public:
  std::vector<psg_layer_desc> layers;

  int index(const std::string& name) const {
    for (std::size_t i = 0; i < layers.size(); ++i)
      if (name == layers[i].name) return static_cast<int>(i);
    throw std::invalid_argument("net: unknown layer '" + name + "'");
  }

  psg_layer_desc& add(int kind, const std::string& name, std::vector<std::string> inputs) {
    if (name.size() >= sizeof(psg_layer_desc{}.name))
      throw std::invalid_argument("net: layer name too long '" + name + "'");
    if (inputs.size() > 8) throw std::invalid_argument("net: too many inputs at '" + name + "'");
    psg_layer_desc d;
    psg_layer_desc_init(&d, kind, name.c_str());
    d.n_inputs = static_cast<int>(inputs.size());
    for (std::size_t i = 0; i < inputs.size(); ++i) d.inputs[i] = index(inputs[i]);
    layers.push_back(d);
    return layers.back();
  }

  void data(const std::string& name, std::size_t b, std::size_t c, std::size_t h,
            std::size_t w) {
    psg_layer_desc& d = add(PSG_LAYER_DATA, name, {});
    d.batch = static_cast<int>(b);
    d.channels = static_cast<int>(c);
    d.height = static_cast<int>(h);
    d.width = static_cast<int>(w);
  }
  void label(const std::string& name, std::size_t b) {
    add(PSG_LAYER_LABEL, name, {}).batch = static_cast<int>(b);
  }
  // Caffe-style bias multipliers (lr_mult 2, decay_mult bias_decay) as in the prototxts
  void conv(const std::string& name, const std::string& in, int k, int filters, int stride = 1,
            int pad = 0, int group = 1, double bias_decay = 1.0) {
    psg_layer_desc& d = add(PSG_LAYER_CONV, name, {in});
    d.kernel_h = d.kernel_w = k;
    d.num_output = filters;
    d.stride_h = d.stride_w = stride;
    d.pad_h = d.pad_w = pad;
    d.group = group;
    d.lr_mult_b = 2.0;
    d.decay_mult_b = bias_decay;
  }
  void pool(const std::string& name, const std::string& in, int k, int stride,
            int method = PSG_POOL_MAX, int pad = 0, bool ceil_mode = true) {
    psg_layer_desc& d = add(PSG_LAYER_POOL, name, {in});
    d.kernel_h = d.kernel_w = k;
    d.stride_h = d.stride_w = stride;
    d.pool = method;
    d.pad_h = d.pad_w = pad;
    d.ceil_mode = ceil_mode ? 1 : 0;
  }
  void linear(const std::string& name, const std::string& in, int outputs,
              double bias_decay = 1.0) {
    psg_layer_desc& d = add(PSG_LAYER_LINEAR, name, {in});
    d.num_output = outputs;
    d.lr_mult_b = 2.0;
    d.decay_mult_b = bias_decay;
  }
  void relu(const std::string& name, const std::string& in) { add(PSG_LAYER_RELU, name, {in}); }
  void lrn(const std::string& name, const std::string& in, int size, double alpha, double beta) {
    psg_layer_desc& d = add(PSG_LAYER_LRN, name, {in});
    d.local_size = size;
    d.alpha = alpha;
    d.beta = beta;
    d.k = 1.0;
  }
  void dropout(const std::string& name, const std::string& in, double ratio) {
    add(PSG_LAYER_DROPOUT, name, {in}).dropout_ratio = ratio;
  }
  void concat(const std::string& name, std::vector<std::string> ins) {
    add(PSG_LAYER_CONCAT, name, std::move(ins));
  }
  void softmax(const std::string& name, const std::string& logits, double weight = 1.0) {
    add(PSG_LAYER_SOFTMAX_LOSS, name, {logits, "label"}).loss_weight = weight;
  }
};

/// Caffe examples/cifar10/cifar10_quick_train_test.prototxt (BASELINE.json configs[0-1]).
inline std::vector<psg_layer_desc> make_cifar10_quick(std::size_t batch, int classes = 10,
                                                      std::size_t c = 3, std::size_t h = 32,
                                                      std::size_t w = 32) {
  DescBuilder n;
  n.data("data", batch, c, h, w);
  n.label("label", batch);
  n.conv("conv1", "data", 5, 32, 1, 2);
  n.pool("pool1", "conv1", 3, 2, PSG_POOL_MAX);
  n.relu("relu1", "pool1");
  n.conv("conv2", "relu1", 5, 32, 1, 2);
  n.relu("relu2", "conv2");
  n.pool("pool2", "relu2", 3, 2, PSG_POOL_AVE);
  n.conv("conv3", "pool2", 5, 64, 1, 2);
  n.relu("relu3", "conv3");
  n.pool("pool3", "relu3", 3, 2, PSG_POOL_AVE);
  n.linear("ip1", "pool3", 64);
  n.linear("ip2", "ip1", classes);
  n.softmax("loss", "ip2");
  return n.layers;
}

/// BVLC AlexNet (models/bvlc_alexnet/train_val.prototxt; BASELINE.json configs[2]).
inline std::vector<psg_layer_desc> make_alexnet(std::size_t batch, int classes = 1000,
                                                std::size_t c = 3, std::size_t h = 227,
                                                std::size_t w = 227) {
  DescBuilder n;
  n.data("data", batch, c, h, w);
  n.label("label", batch);
  n.conv("conv1", "data", 11, 96, 4, 0, 1, 0.0);
  n.relu("relu1", "conv1");
  n.lrn("norm1", "relu1", 5, 1e-4, 0.75);
  n.pool("pool1", "norm1", 3, 2);
  n.conv("conv2", "pool1", 5, 256, 1, 2, 2, 0.0);
  n.relu("relu2", "conv2");
  n.lrn("norm2", "relu2", 5, 1e-4, 0.75);
  n.pool("pool2", "norm2", 3, 2);
  n.conv("conv3", "pool2", 3, 384, 1, 1, 1, 0.0);
  n.relu("relu3", "conv3");
  n.conv("conv4", "relu3", 3, 384, 1, 1, 2, 0.0);
  n.relu("relu4", "conv4");
  n.conv("conv5", "relu4", 3, 256, 1, 1, 2, 0.0);
  n.relu("relu5", "conv5");
  n.pool("pool5", "relu5", 3, 2);
  n.linear("fc6", "pool5", 4096, 0.0);
  n.relu("relu6", "fc6");
  n.dropout("drop6", "relu6", 0.5);
  n.linear("fc7", "drop6", 4096, 0.0);
  n.relu("relu7", "fc7");
  n.dropout("drop7", "relu7", 0.5);
  n.linear("fc8", "drop7", classes, 0.0);
  n.softmax("loss", "fc8");
  return n.layers;
}

namespace detail {

inline std::string inception(DescBuilder& n, const std::string& name, const std::string& in,
                             int c1, int c3r, int c3, int c5r, int c5, int cp) {
  const std::string p = name + "/";
  n.conv(p + "1x1", in, 1, c1, 1, 0, 1, 0.0);
  n.relu(p + "relu_1x1", p + "1x1");
  n.conv(p + "3x3_reduce", in, 1, c3r, 1, 0, 1, 0.0);
  n.relu(p + "relu_3x3_reduce", p + "3x3_reduce");
  n.conv(p + "3x3", p + "relu_3x3_reduce", 3, c3, 1, 1, 1, 0.0);
  n.relu(p + "relu_3x3", p + "3x3");
  n.conv(p + "5x5_reduce", in, 1, c5r, 1, 0, 1, 0.0);
  n.relu(p + "relu_5x5_reduce", p + "5x5_reduce");
  n.conv(p + "5x5", p + "relu_5x5_reduce", 5, c5, 1, 2, 1, 0.0);
  n.relu(p + "relu_5x5", p + "5x5");
  n.pool(p + "pool", in, 3, 1, PSG_POOL_MAX, 1);
  n.conv(p + "pool_proj", p + "pool", 1, cp, 1, 0, 1, 0.0);
  n.relu(p + "relu_pool_proj", p + "pool_proj");
  n.concat(p + "output", {p + "relu_1x1", p + "relu_3x3", p + "relu_5x5", p + "relu_pool_proj"});
  return p + "output";
}

inline void aux_head(DescBuilder& n, const std::string& name, const std::string& in,
                     int classes) {
  const std::string p = name + "/";
  n.pool(p + "ave_pool", in, 5, 3, PSG_POOL_AVE);
  n.conv(p + "conv", p + "ave_pool", 1, 128, 1, 0, 1, 0.0);
  n.relu(p + "relu_conv", p + "conv");
  n.linear(p + "fc", p + "relu_conv", 1024, 0.0);
  n.relu(p + "relu_fc", p + "fc");
  n.dropout(p + "drop_fc", p + "relu_fc", 0.7);
  n.linear(p + "classifier", p + "drop_fc", classes, 0.0);
  n.softmax(p + "loss", p + "classifier", 0.3);
}

}  // namespace detail

/// Caffe bvlc_googlenet with both auxiliary heads (loss weight 0.3; BASELINE.json configs[3]).
inline std::vector<psg_layer_desc> make_googlenet(std::size_t batch, int classes = 1000,
                                                  std::size_t c = 3, std::size_t image = 224) {
  DescBuilder n;
  n.data("data", batch, c, image, image);
  n.label("label", batch);
  n.conv("conv1/7x7_s2", "data", 7, 64, 2, 3, 1, 0.0);
  n.relu("conv1/relu_7x7", "conv1/7x7_s2");
  n.pool("pool1/3x3_s2", "conv1/relu_7x7", 3, 2);
  n.lrn("pool1/norm1", "pool1/3x3_s2", 5, 1e-4, 0.75);
  n.conv("conv2/3x3_reduce", "pool1/norm1", 1, 64, 1, 0, 1, 0.0);
  n.relu("conv2/relu_3x3_reduce", "conv2/3x3_reduce");
  n.conv("conv2/3x3", "conv2/relu_3x3_reduce", 3, 192, 1, 1, 1, 0.0);
  n.relu("conv2/relu_3x3", "conv2/3x3");
  n.lrn("conv2/norm2", "conv2/relu_3x3", 5, 1e-4, 0.75);
  n.pool("pool2/3x3_s2", "conv2/norm2", 3, 2);
  std::string x = detail::inception(n, "inception_3a", "pool2/3x3_s2", 64, 96, 128, 16, 32, 32);
  x = detail::inception(n, "inception_3b", x, 128, 128, 192, 32, 96, 64);
  n.pool("pool3/3x3_s2", x, 3, 2);
  x = detail::inception(n, "inception_4a", "pool3/3x3_s2", 192, 96, 208, 16, 48, 64);
  detail::aux_head(n, "loss1", x, classes);
  x = detail::inception(n, "inception_4b", x, 160, 112, 224, 24, 64, 64);
  x = detail::inception(n, "inception_4c", x, 128, 128, 256, 24, 64, 64);
  x = detail::inception(n, "inception_4d", x, 112, 144, 288, 32, 64, 64);
  detail::aux_head(n, "loss2", x, classes);
  x = detail::inception(n, "inception_4e", x, 256, 160, 320, 32, 128, 128);
  n.pool("pool4/3x3_s2", x, 3, 2);
  x = detail::inception(n, "inception_5a", "pool4/3x3_s2", 256, 160, 320, 32, 128, 128);
  x = detail::inception(n, "inception_5b", x, 384, 192, 384, 48, 128, 128);
  n.pool("pool5/7x7_s1", x, 7, 1, PSG_POOL_AVE, 0, false);
  n.dropout("pool5/drop_7x7_s1", "pool5/7x7_s1", 0.4);
  n.linear("loss3/classifier", "pool5/drop_7x7_s1", classes, 0.0);
  n.softmax("loss3/loss3", "loss3/classifier");
  return n.layers;
}

/// `net.preset` extension values (config keys, parasgd_b200/experiment.hpp).
inline bool is_caffe_preset(const std::string& name) {
  return name == "cifar10_quick" || name == "alexnet" || name == "googlenet";
}

inline std::vector<psg_layer_desc> caffe_preset(const std::string& name, std::size_t batch,
                                                std::size_t c, std::size_t h, std::size_t w,
                                                int classes) {
  if (name == "cifar10_quick") return make_cifar10_quick(batch, classes, c, h, w);
  if (name == "alexnet") return make_alexnet(batch, classes, c, h, w);
  if (name == "googlenet") {
    if (h != w) throw std::invalid_argument("googlenet: square images only");
    return make_googlenet(batch, classes, c, h);
  }
  throw std::invalid_argument("unknown preset '" + name + "'");
}

}  // namespace b200
}  // namespace parasgd
