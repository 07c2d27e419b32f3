"""B200-native V(s) scoring path for the `tensched` greedy value-function
scheduler (arXiv 2011.14486): bit-exact loop-nest featurization, LSTM value
network and fused per-layer argmin on sm_100a, behind the reference's
scheduler/value-function API."""

__version__ = "0.1.0"
