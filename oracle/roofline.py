"""Arithmetic-intensity closed forms (oracle; test infrastructure only).

Table tab:arithmetic-intensity and the general form P:133-140.
"""


def ai_closed_form(variant, L, h_q, g_q=None, m_kv=None):
    """Evaluate the Table-1 column for ``variant`` at KV length L."""
    if variant == "GLA-2":
        return L / (1 + L / h_q)
    if variant == "GLA":
        return L / (1 + L / (2 * g_q))
    if variant == "MLA":
        return L / (1 + L / (2 * h_q))
    if variant == "MQA":
        return L * h_q / (h_q + L)
    if variant == "GQA":
        return L * h_q / (h_q + (h_q / g_q) * L)
    if variant == "GTA":
        return 2 * L * h_q / (2 * h_q + (h_q / g_q) * L)
    if variant == "MHA":
        return L / (1 + L)
    if variant == "General":
        return 2 * L / (2 + (m_kv / g_q) * L)
    raise ValueError(variant)


def ai_asymptote(variant, h_q, g_q=None, m_kv=None):
    """Second row of Table 1 (L >> h_q)."""
    return {
        "GLA-2": h_q, "GLA": 2 * g_q if g_q else None, "MLA": 2 * h_q, "MQA": h_q,
        "GQA": g_q, "GTA": 2 * g_q if g_q else None, "MHA": 1,
        "General": 2 * g_q / m_kv if (g_q and m_kv) else None,
    }[variant]
