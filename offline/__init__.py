"""Host-side offline stage of LRBMS: the local reduced bases Phi_E (a shared input of the online step)."""
