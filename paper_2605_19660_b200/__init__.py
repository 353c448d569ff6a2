"""B200-native OScaR KV-cache path (quantize/append + fused-dequant split-KV
decode attention) behind the reference's KvCache API.  See DESIGN.md."""
from .kv_cache import DecodeBatch, KvCache, PipelineConfig, lse_merge  # noqa: F401

__all__ = ["DecodeBatch", "KvCache", "PipelineConfig", "lse_merge"]
