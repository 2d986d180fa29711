"""paper_2403_13135_b200: B200-native (sm_100a) sea-ice auto-labeling and U-Net training.

Drop-in for the hot paths of the arxiv 2403.13135 reference:
  * icelabel.process_tile / apply_filter / segment  -> fused CUDA kernel K1 / K1s
  * icetrain.UNet / synchronized_step / train_distributed -> tcgen05 conv kernels + NCCL DP
"""
__version__ = "0.1.0"
