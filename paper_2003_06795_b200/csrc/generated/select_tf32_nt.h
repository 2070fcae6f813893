#ifndef SELECT_TF32_NT_H
#define SELECT_TF32_NT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_nt_config;

static inline select_tf32_nt_config select_tf32_nt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(3584)) {
        if (n < INT64_C(2897)) {
            if (n < INT64_C(444)) {
                if (n < INT64_C(46)) {
                    if (m < INT64_C(2218)) {
                        if (m < INT64_C(1109)) {
                            select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(167)) {
                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(167)) {
                            select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (k < INT64_C(992)) {
                        if (m < INT64_C(1109)) {
                            if (m < INT64_C(112)) {
                                if (m < INT64_C(80)) {
                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(744)) {
                                        select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(544)) {
                                    if (k < INT64_C(314)) {
                                        select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(79)) {
                                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(278)) {
                                                if (k < INT64_C(444)) {
                                                    select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (n < INT64_C(182)) {
                                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (n < INT64_C(79)) {
                                if (m < INT64_C(2218)) {
                                    select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(314)) {
                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(2218)) {
                                        select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(1087)) {
                            if (m < INT64_C(555)) {
                                if (m < INT64_C(278)) {
                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(2218)) {
                                    select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(2218)) {
                                select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(182)) {
                                    select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(1268)) {
                    if (m < INT64_C(634)) {
                        if (k < INT64_C(2897)) {
                            if (m < INT64_C(3)) {
                                if (m < INT64_C(2)) {
                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(1145)) {
                                    if (m < INT64_C(139)) {
                                        if (m < INT64_C(70)) {
                                            if (m < INT64_C(12)) {
                                                select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(29)) {
                                                    if (k < INT64_C(1620)) {
                                                        select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(405)) {
                                                select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(725)) {
                                        if (m < INT64_C(278)) {
                                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(139)) {
                                            select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(3)) {
                                if (m < INT64_C(2)) {
                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(70)) {
                                    select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(278)) {
                                        select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(144)) {
                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(2173)) {
                                if (m < INT64_C(896)) {
                                    if (k < INT64_C(405)) {
                                        if (k < INT64_C(287)) {
                                            select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(544)) {
                        if (m < INT64_C(2218)) {
                            if (k < INT64_C(544)) {
                                select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(363)) {
                            select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(2218)) {
                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            }
        } else {
            if (k < INT64_C(10138)) {
                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                return out;
            } else {
                select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                return out;
            }
        }
    } else {
        if (k < INT64_C(815)) {
            if (m < INT64_C(17740)) {
                if (n < INT64_C(222)) {
                    if (n < INT64_C(91)) {
                        if (k < INT64_C(222)) {
                            if (k < INT64_C(146)) {
                                if (n < INT64_C(46)) {
                                    if (k < INT64_C(118)) {
                                        select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(8870)) {
                                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(28)) {
                                                select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (n < INT64_C(167)) {
                            select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(8870)) {
                                select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                }
            } else {
                if (k < INT64_C(384)) {
                    if (m < INT64_C(35480)) {
                        if (n < INT64_C(46)) {
                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (n < INT64_C(91)) {
                        if (m < INT64_C(35480)) {
                            select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(567677)) {
                                select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(35480)) {
                            select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(363)) {
                if (m < INT64_C(35480)) {
                    if (m < INT64_C(17740)) {
                        if (m < INT64_C(8870)) {
                            if (k < INT64_C(1630)) {
                                select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(182)) {
                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                    return out;
                }
            } else {
                select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_TF32_NT_H */
