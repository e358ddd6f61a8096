// Paper U-Net state shared by the inference (hb_paper.cu) and training
// (hb_train.cu) paths: the parameter registry in the reference's names and
// creation order (NetworkWeights, inc/unet.hpp:10-111) and the device copies.
#pragma once
#include <map>
#include <string>
#include <vector>

#include "hb_internal.h"

namespace hb {

struct PParam {
  std::string name;
  int d[4];
  std::vector<float> v;
  size_t size() const { return size_t(d[0]) * d[1] * d[2] * d[3]; }
};

// one tensor-core implicit GEMM of a paper-net convolution: the whole conv, or
// one output parity class of a stride-2 transposed conv (hb_conv_tc.cu)
struct PaperTc {
  ConvW cw;  // dwh / dwl [cout][ntaps * cin] (3xTF32 split), db bias; cout padded to a multiple of 16
  TcGeo geo; // taps, input origin offsets; output class (py, px)
  DBuf<float> mu, is, g, be;  // batch-norm buffers padded like cout (when the conv has one)
};

struct DevConv {  // one convolution with its fused epilogue
  int cout = 0, cin = 0, k = 0;
  bool transpose = false, bn = false;
  DBuf<float> w, bias, mu, is, g, be;
  std::vector<float> hw, hb;  // host copies of w ([tap][cin][cout]) and bias: the 16 -> 2 head's kernel parameters
  std::vector<PaperTc> tc;  // tensor-core form (empty: channels not multiples of 16)
};

struct PaperState {
  hb_unet_cfg cfg{};
  int variant = 0;  // 0 standalone ("unet."), 1 encoder_solver ("enc." + "sol.")
  bool active = false;
  std::vector<PParam> params;  // registry order
  std::map<std::string, size_t> index;
  std::map<std::string, DevConv> dev;  // by kernel name
  bool dirty = true;
  bool par4 = true;  // stride-2 transposed convs as ONE 4-parity-class GEMM (else four class launches)
  unsigned long long host_gen = 0;  // bumped when the host parameters change from outside training
  // encoder features (batch 1), per level
  std::vector<DBuf<float>> feat;
  unsigned long long feat_gen = ~0ull;
  DBuf<float> k2f, gamf;  // fine-level kappa^2 and gamma (fp32) for the input stack
  unsigned long long coef_gen = ~0ull;
  DBuf<float> arena, io;
};

// the context's paper-net state (created on first use)
PaperState& paper_state(Context& c);

}  // namespace hb
