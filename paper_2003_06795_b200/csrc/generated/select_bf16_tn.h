#ifndef SELECT_BF16_TN_H
#define SELECT_BF16_TN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_bf16_tn_config;

static inline select_bf16_tn_config select_bf16_tn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(17740)) {
        if (m < INT64_C(2218)) {
            if (n < INT64_C(744)) {
                if (k < INT64_C(992)) {
                    if (m < INT64_C(224)) {
                        if (m < INT64_C(112)) {
                            if (n < INT64_C(227)) {
                                if (k < INT64_C(193)) {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(111)) {
                                if (n < INT64_C(79)) {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(471)) {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(222)) {
                            if (m < INT64_C(1109)) {
                                if (k < INT64_C(46)) {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(444)) {
                                        if (n < INT64_C(46)) {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(555)) {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(111)) {
                                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (n < INT64_C(46)) {
                                    if (k < INT64_C(167)) {
                                        select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(544)) {
                                if (m < INT64_C(317)) {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    if (m < INT64_C(634)) {
                                        if (n < INT64_C(79)) {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (n < INT64_C(111)) {
                                            if (m < INT64_C(1109)) {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (n < INT64_C(79)) {
                                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(363)) {
                                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(1109)) {
                                                    if (n < INT64_C(182)) {
                                                        select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    if (n < INT64_C(182)) {
                                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(1109)) {
                                    if (m < INT64_C(555)) {
                                        if (n < INT64_C(124)) {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(139)) {
                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(1537)) {
                            if (n < INT64_C(363)) {
                                if (k < INT64_C(1087)) {
                                    if (m < INT64_C(278)) {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(555)) {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(1109)) {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(278)) {
                                select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                if (k < INT64_C(2173)) {
                                    select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(3259)) {
                                        if (m < INT64_C(1109)) {
                                            if (n < INT64_C(363)) {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(555)) {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(555)) {
                    if (m < INT64_C(3)) {
                        if (k < INT64_C(1620)) {
                            select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(2897)) {
                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(2)) {
                                    if (n < INT64_C(2024)) {
                                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(1620)) {
                            if (k < INT64_C(1620)) {
                                if (m < INT64_C(139)) {
                                    if (k < INT64_C(227)) {
                                        if (m < INT64_C(70)) {
                                            select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(287)) {
                                        if (m < INT64_C(278)) {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(203)) {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(278)) {
                                            if (k < INT64_C(405)) {
                                                select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(6)) {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(12)) {
                                        select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(2897)) {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(12)) {
                                if (k < INT64_C(10138)) {
                                    select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(278)) {
                                    if (m < INT64_C(70)) {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(139)) {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(405)) {
                        if (m < INT64_C(1109)) {
                            if (k < INT64_C(203)) {
                                select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(287)) {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(725)) {
                            select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(896)) {
                                select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(444)) {
                if (n < INT64_C(111)) {
                    if (k < INT64_C(146)) {
                        if (k < INT64_C(42)) {
                            select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(8870)) {
                                if (k < INT64_C(79)) {
                                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(4435)) {
                                        select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(118)) {
                                            select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (n < INT64_C(46)) {
                            select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(79)) {
                                if (k < INT64_C(471)) {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(8870)) {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(4435)) {
                        if (n < INT64_C(167)) {
                            if (k < INT64_C(544)) {
                                select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(46)) {
                                select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(725)) {
                                    select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(1630)) {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(222)) {
                            if (m < INT64_C(8870)) {
                                if (k < INT64_C(91)) {
                                    select_bf16_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(363)) {
                                        select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(8870)) {
                                if (k < INT64_C(272)) {
                                    select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (k < INT64_C(1087)) {
                    if (k < INT64_C(111)) {
                        select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(3584)) {
                        select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(3072)) {
                            if (m < INT64_C(8870)) {
                                select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_tn_config out = {4u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        } else {
                            select_bf16_tn_config out = {4u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            }
        }
    } else {
        if (k < INT64_C(815)) {
            if (n < INT64_C(46)) {
                if (m < INT64_C(35480)) {
                    select_bf16_tn_config out = {4u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (k < INT64_C(68)) {
                        select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_tn_config out = {4u, 1u, 1u, 16u, 16u};
                        return out;
                    }
                }
            } else {
                if (k < INT64_C(384)) {
                    select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                } else {
                    if (n < INT64_C(91)) {
                        if (m < INT64_C(35480)) {
                            select_bf16_tn_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(70960)) {
                            select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_tn_config out = {4u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (m < INT64_C(35480)) {
                select_bf16_tn_config out = {1u, 1u, 2u, 8u, 8u};
                return out;
            } else {
                select_bf16_tn_config out = {4u, 1u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_BF16_TN_H */
