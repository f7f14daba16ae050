#!/usr/bin/env bash
# Mutation check for the oracle's pins: each mutation is a plausible mistake in
# oracle/cce_oracle.c; the pin suite must fail for every one of them.
set -u
cd "$(dirname "$0")/.."
cp oracle/cce_oracle.c /tmp/oracle_orig.c
trap 'cp /tmp/oracle_orig.c oracle/cce_oracle.c; python -c "import oracle; oracle.build(force=True)"' EXIT
muts=(
 's/double ce = p - (is_target ? 1.0 : 0.0);/double ce = p;/'            # dropped one-hot
 's/dloss \/ (double)nv/dloss \/ (double)N/'                           # wrong mean divisor
 's/for (int64_t v = 0; v < V; ++v) s += exp(z\[v\] - m);/for (int64_t v = 1; v < V; ++v) s += exp(z[v] - m);/'  # dropped term
 's/out\[d\] += g \* hr\[d\];/out[d] += g * w[d];/'                   # transposed operand in dW
 's/row_loss\[n\] = (1.0 - eps) \* (l - z\[y\])/row_loss[n] = (1.0 - eps) * (l + z[y])/'  # sign
 's/return m + log(s);/return log(s);/'                                # dropped max shift
 's/double g = rscale\[n\] \* row_grad(zv, lse\[n\]/double g = rscale[n] * row_grad(zv, lse[0]/'  # wrong index
 's/return (1.0 - eps) \* ce + eps \* uni + zl;/return (1.0 - eps) * (ce + zl) + eps * uni;/'  # z-loss grad blended (Liger order)
 's/+ lam \* l \* l;/+ (1.0 - eps) * lam * l * l;/'                  # z-loss term blended (Liger order)
 's/double uni = p - 1.0 \/ (double)V;/double uni = p - 1.0 \/ (double)(V - 1);/'  # wrong uniform mass
 's/eps \* (l - zsum \/ (double)V)/eps * (l - zsum \/ (double)(V + 1))/'  # wrong mean of logits
 's/double zl = 2.0 \* lam \* lse \* p;/double zl = lam * lse * p;/'  # dropped factor 2
 's/(reduction == 1 ? dloss : (dloss_rows ? dloss_rows\[n\]/(reduction == 1 ? dloss \/ (double)nv : (dloss_rows ? dloss_rows[n]/'  # sum divided by n_valid
 's/(dloss_rows ? dloss_rows\[n\] : 0.0)/(dloss_rows ? dloss_rows[0] : 0.0)/'  # none: wrong row of dloss
 's/loss\[n\] = labels\[n\] != ignore_index ? row_loss\[n\] : 0.0;/loss[n] = labels[n] != ignore_index ? row_loss[n] \/ (double)nv : 0.0;/'  # none: per-row loss averaged
)
# fused AdamW (oracle_adamw_step)
muts+=(
 's/double th = theta\[i\] \* (1.0 - lr \* wd);/double th = theta[i];/'           # dropped weight decay
 's/double g = grad\[i\] \* clip_coef;/double g = grad[i];/'                    # dropped clipping
 's/double vh = v\[i\] \/ bc2;/double vh = v[i];/'                                # dropped bias correction
 's/theta\[i\] = th - lr \* (mh \/ (sqrt(vh) + eps));/theta[i] = th - lr * (mh \/ sqrt(vh + eps));/'  # eps inside sqrt
)
# RMSNorm prologue (oracle_rmsnorm_fwd / _bwd)
muts+=(
 's/const double r = sqrt(ss \/ (double)D + eps);/const double r = sqrt(ss + eps);/'          # dropped 1\/D (the Prop. garble)
 's/for (int64_t k = 0; k < D; ++k) dxr\[k\] = rs \* (gamma\[k\] \* dyr\[k\] - (xr\[k\] \* rs) \* c1);/for (int64_t k = 0; k < D; ++k) dxr[k] = rs * gamma[k] * (dyr[k] - (xr[k] * rs) * c1);/'  # gamma on both terms (the Alg. garble)
 's/c1 \/= (double)D;/c1 \/= 1.0;/'                                                       # dropped mean in c1
 's/dgamma\[k\] += dyr\[k\] \* (xr\[k\] \* rs);/dgamma[k] += dyr[k] * xr[k];/'           # dgamma without rstd
)
# bf16 rounding (oracle_to_bf16)
muts+=(
 's/u += 0x7FFFu + ((u >> 16) \& 1u);/u += 0u;/'                         # truncation
 's/u += 0x7FFFu + ((u >> 16) \& 1u);/u += 0x8000u;/'                    # ties away from zero
 's/u += 0x7FFFu + ((u >> 16) \& 1u);/u += 0x7FFFu + (((u >> 16) \& 1u) ^ 1u);/'  # ties to odd
 's/if ((u \& 0x7FFFFFFFu) > 0x7F800000u) {/if (0) {/'  # NaN branch dropped
)
fail=0
for m in "${muts[@]}"; do
  cp /tmp/oracle_orig.c oracle/cce_oracle.c
  sed -i "$m" oracle/cce_oracle.c
  if cmp -s /tmp/oracle_orig.c oracle/cce_oracle.c; then echo "NO-OP mutation: $m"; fail=1; continue; fi
  python -c "import oracle; oracle.build(force=True)"
  if python -m pytest tests/test_oracle_pins.py -q -x >/dev/null 2>&1; then
    echo "SURVIVED: $m"; fail=1
  else
    echo "killed:   $m"
  fi
done
exit $fail
