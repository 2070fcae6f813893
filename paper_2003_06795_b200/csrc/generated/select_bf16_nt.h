#ifndef SELECT_BF16_NT_H
#define SELECT_BF16_NT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_bf16_nt_config;

static inline select_bf16_nt_config select_bf16_nt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(4435)) {
        if (k < INT64_C(3072)) {
            if (n < INT64_C(79)) {
                if (k < INT64_C(118)) {
                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (k < INT64_C(471)) {
                        if (k < INT64_C(222)) {
                            if (k < INT64_C(167)) {
                                if (m < INT64_C(1109)) {
                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(2218)) {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(314)) {
                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(555)) {
                                    if (m < INT64_C(278)) {
                                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (m < INT64_C(634)) {
                    if (n < INT64_C(1012)) {
                        if (m < INT64_C(70)) {
                            if (m < INT64_C(12)) {
                                if (m < INT64_C(6)) {
                                    if (m < INT64_C(2)) {
                                        if (k < INT64_C(1620)) {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(3)) {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(1620)) {
                                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(405)) {
                                    if (n < INT64_C(227)) {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (n < INT64_C(744)) {
                                if (k < INT64_C(314)) {
                                    if (k < INT64_C(79)) {
                                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(744)) {
                                        if (m < INT64_C(139)) {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(444)) {
                                                if (m < INT64_C(278)) {
                                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(139)) {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(278)) {
                                                if (k < INT64_C(2173)) {
                                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (n < INT64_C(287)) {
                                                    if (k < INT64_C(992)) {
                                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (k < INT64_C(1536)) {
                                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    }
                                                } else {
                                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                }
                            } else {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(278)) {
                            if (k < INT64_C(287)) {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(70)) {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(139)) {
                                        if (k < INT64_C(725)) {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(725)) {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (n < INT64_C(544)) {
                        if (n < INT64_C(363)) {
                            if (k < INT64_C(1630)) {
                                if (n < INT64_C(222)) {
                                    if (k < INT64_C(544)) {
                                        if (m < INT64_C(2218)) {
                                            if (n < INT64_C(111)) {
                                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(1109)) {
                                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(91)) {
                                                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (k < INT64_C(363)) {
                                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    }
                                                }
                                            }
                                        } else {
                                            if (n < INT64_C(111)) {
                                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(1109)) {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(2218)) {
                                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(2218)) {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(725)) {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(1087)) {
                                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(1109)) {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(2218)) {
                                if (k < INT64_C(1449)) {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(1109)) {
                                        select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(1268)) {
                            if (n < INT64_C(1620)) {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(1025)) {
                                if (m < INT64_C(2218)) {
                                    if (k < INT64_C(222)) {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                }
            }
        } else {
            if (k < INT64_C(10752)) {
                if (m < INT64_C(12)) {
                    select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                } else {
                    if (m < INT64_C(278)) {
                        if (m < INT64_C(40)) {
                            if (n < INT64_C(2024)) {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(2218)) {
                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(3)) {
                    select_bf16_nt_config out = {8u, 1u, 8u, 16u, 16u};
                    return out;
                } else {
                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                    return out;
                }
            }
        }
    } else {
        if (k < INT64_C(815)) {
            if (m < INT64_C(17740)) {
                if (n < INT64_C(79)) {
                    if (k < INT64_C(46)) {
                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(385)) {
                            if (m < INT64_C(8870)) {
                                if (n < INT64_C(28)) {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(167)) {
                                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(222)) {
                                            select_bf16_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (k < INT64_C(222)) {
                                    if (k < INT64_C(118)) {
                                        if (k < INT64_C(79)) {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (n < INT64_C(46)) {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(8870)) {
                        if (k < INT64_C(64)) {
                            if (k < INT64_C(28)) {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(363)) {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (n < INT64_C(28)) {
                    if (m < INT64_C(35480)) {
                        if (k < INT64_C(118)) {
                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (n < INT64_C(111)) {
                        select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(70960)) {
                            select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nt_config out = {8u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (m < INT64_C(7168)) {
                if (k < INT64_C(3259)) {
                    if (n < INT64_C(182)) {
                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    select_bf16_nt_config out = {8u, 1u, 8u, 16u, 16u};
                    return out;
                }
            } else {
                if (m < INT64_C(35480)) {
                    if (k < INT64_C(1630)) {
                        if (m < INT64_C(17740)) {
                            if (n < INT64_C(182)) {
                                select_bf16_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_bf16_nt_config out = {8u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                } else {
                    select_bf16_nt_config out = {8u, 1u, 8u, 16u, 16u};
                    return out;
                }
            }
        }
    }
}

#endif /* SELECT_BF16_NT_H */
