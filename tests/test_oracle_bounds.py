"""Pins of the Bayesian lower bound ℓ_α = I^{-1}(1 − α; 1 + TP, 1 + FN) (Eqs. recall/precision
lower bound; Q7) used by the host derivations: closed forms and values."""
import math

import pytest

import oracle


def test_flat_prior_no_data():
    # Beta(1,1) = uniform: the 5 % quantile is 0.05
    assert abs(oracle.beta_lower_bound(0, 0, 0.95) - 0.05) < 1e-12


@pytest.mark.parametrize("tp", [0, 1, 5, 19, 200])
def test_no_false_negatives_closed_form(tp):
    # Beta(1+TP, 1): CDF x^(1+TP) ⇒ ℓ = (1 − α)^(1/(1+TP))
    assert abs(oracle.beta_lower_bound(tp, 0, 0.95) - 0.05 ** (1.0 / (1 + tp))) < 1e-12


@pytest.mark.parametrize("fn", [0, 3, 9, 100])
def test_no_true_positives_closed_form(fn):
    # Beta(1, 1+FN): CDF 1 − (1−x)^(1+FN) ⇒ ℓ = 1 − α^(1/(1+FN))
    assert abs(oracle.beta_lower_bound(0, fn, 0.95) - (1 - 0.95 ** (1.0 / (1 + fn)))) < 1e-12


def test_survey_values_and_monotonicity():
    assert abs(oracle.beta_lower_bound(19, 0, 0.95) - 0.8608916593) < 1e-9
    assert abs(oracle.beta_lower_bound(19, 1, 0.95) - 0.7932746210) < 1e-9
    assert abs(oracle.beta_lower_bound(90, 10, 0.95) - 0.8378454281) < 1e-9
    assert abs(oracle.beta_lower_bound(900, 100, 0.95) - 0.8831242356) < 1e-9
    # more TP raises, more FN lowers, higher credibility lowers the bound
    assert oracle.beta_lower_bound(50, 5, 0.95) > oracle.beta_lower_bound(40, 5, 0.95)
    assert oracle.beta_lower_bound(50, 5, 0.95) > oracle.beta_lower_bound(50, 6, 0.95)
    assert oracle.beta_lower_bound(50, 5, 0.99) < oracle.beta_lower_bound(50, 5, 0.9)
