EE_GEMM_CTA=1 python scripts/trace_gemm.py
EE_GEMM_CTA=1 EE_GEMM_CLUSTER=2 python scripts/trace_gemm.py
EE_GEMM_CTA=2 python scripts/trace_gemm.py
